// jf_k_gauss2d_x2.cu — pass-kernel instances for ModelGauss2DRotX2 (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
Kernels kernels_gauss2d_x2(int coord) {
  if (coord == COORD_EXPLICIT) return Kernels{pass_kernel<ModelGauss2DRotX2, true, COORD_EXPLICIT>, pass_kernel<ModelGauss2DRotX2, false, COORD_EXPLICIT>};
  return Kernels{pass_kernel<ModelGauss2DRotX2, true, COORD_GRID>, pass_kernel<ModelGauss2DRotX2, false, COORD_GRID>};
}
}  // namespace jf

// jf_k_gauss2d.cu — pass-kernel instances for ModelGauss2DRot (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
Kernels kernels_gauss2d(int coord) {
  if (coord == COORD_EXPLICIT) return Kernels{pass_kernel<ModelGauss2DRot, true, COORD_EXPLICIT>, pass_kernel<ModelGauss2DRot, false, COORD_EXPLICIT>};
  return Kernels{pass_kernel<ModelGauss2DRot, true, COORD_GRID>, pass_kernel<ModelGauss2DRot, false, COORD_GRID>};
}
}  // namespace jf

// jf_k_gauss1d.cu — pass-kernel instances for ModelGauss1D (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
Kernels kernels_gauss1d(int coord) {
  if (coord == COORD_EXPLICIT) return Kernels{pass_kernel<ModelGauss1D, true, COORD_EXPLICIT>, pass_kernel<ModelGauss1D, false, COORD_EXPLICIT>};
  return Kernels{pass_kernel<ModelGauss1D, true, COORD_IMPLICIT_T>, pass_kernel<ModelGauss1D, false, COORD_IMPLICIT_T>};
}
}  // namespace jf

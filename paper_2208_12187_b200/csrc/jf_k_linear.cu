// jf_k_linear.cu — pass-kernel instances for ModelLinear (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
Kernels kernels_linear(int coord) {
  if (coord == COORD_EXPLICIT) return Kernels{pass_kernel<ModelLinear, true, COORD_EXPLICIT>, pass_kernel<ModelLinear, false, COORD_EXPLICIT>};
  return Kernels{pass_kernel<ModelLinear, true, COORD_IMPLICIT_T>, pass_kernel<ModelLinear, false, COORD_IMPLICIT_T>};
}
}  // namespace jf

// jf_k_exp_decay.cu — pass-kernel instances for ModelExpDecay (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
Kernels kernels_exp_decay(int coord) {
  if (coord == COORD_EXPLICIT) return Kernels{pass_kernel<ModelExpDecay, true, COORD_EXPLICIT>, pass_kernel<ModelExpDecay, false, COORD_EXPLICIT>};
  return Kernels{pass_kernel<ModelExpDecay, true, COORD_IMPLICIT_T>, pass_kernel<ModelExpDecay, false, COORD_IMPLICIT_T>};
}
}  // namespace jf

// jf_k_exp_decay.cu — pass-kernel instances for ModelExpDecay (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelExpDecay, true, C, false>;
  k.rk = pass_kernel<ModelExpDecay, false, C, false>;
  k.jkw = pass_kernel<ModelExpDecay, true, C, true>;
  k.rkw = pass_kernel<ModelExpDecay, false, C, true>;
  k.jtpb = PassCfg<ModelExpDecay, true>::TPB;
  k.jsplit = PassCfg<ModelExpDecay, true>::SPLIT;
  k.small = fit_small_kernel<ModelExpDecay, C, false>;
  k.batch = fit_batch_kernel<ModelExpDecay, C, false>;
  k.batchw = fit_batch_kernel<ModelExpDecay, C, true>;
  k.smallw = fit_small_kernel<ModelExpDecay, C, true>;
  k.rtpb = PassCfg<ModelExpDecay, false>::TPB;
  return k;
}
Kernels kernels_exp_decay(int coord) { return coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_IMPLICIT_T>(); }
}  // namespace jf

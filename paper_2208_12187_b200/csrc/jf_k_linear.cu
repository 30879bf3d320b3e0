// jf_k_linear.cu — pass-kernel instances for ModelLinear (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelLinear, true, C, false>;
  k.rk = pass_kernel<ModelLinear, false, C, false>;
  k.jkw = pass_kernel<ModelLinear, true, C, true>;
  k.rkw = pass_kernel<ModelLinear, false, C, true>;
  k.jtpb = PassCfg<ModelLinear, true>::TPB;
  k.jsplit = PassCfg<ModelLinear, true>::SPLIT;
  k.small = fit_small_kernel<ModelLinear, C, false>;
  k.batch = fit_batch_kernel<ModelLinear, C, false>;
  k.batchw = fit_batch_kernel<ModelLinear, C, true>;
  k.smallw = fit_small_kernel<ModelLinear, C, true>;
  k.rtpb = PassCfg<ModelLinear, false>::TPB;
  return k;
}
Kernels kernels_linear(int coord) { return coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_IMPLICIT_T>(); }
}  // namespace jf

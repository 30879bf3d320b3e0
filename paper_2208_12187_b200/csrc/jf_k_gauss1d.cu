// jf_k_gauss1d.cu — pass-kernel instances for ModelGauss1D (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelGauss1D, true, C, false>;
  k.rk = pass_kernel<ModelGauss1D, false, C, false>;
  k.jkw = pass_kernel<ModelGauss1D, true, C, true>;
  k.rkw = pass_kernel<ModelGauss1D, false, C, true>;
  k.jtpb = PassCfg<ModelGauss1D, true>::TPB;
  k.jsplit = PassCfg<ModelGauss1D, true>::SPLIT;
  k.small = fit_small_kernel<ModelGauss1D, C, false>;
  k.batch = fit_batch_kernel<ModelGauss1D, C, false>;
  k.batchw = fit_batch_kernel<ModelGauss1D, C, true>;
  k.smallw = fit_small_kernel<ModelGauss1D, C, true>;
  k.rtpb = PassCfg<ModelGauss1D, false>::TPB;
  return k;
}
Kernels kernels_gauss1d(int coord) { return coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_IMPLICIT_T>(); }
}  // namespace jf

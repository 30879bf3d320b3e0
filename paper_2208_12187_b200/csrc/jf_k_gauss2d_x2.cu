// jf_k_gauss2d_x2.cu — pass-kernel instances for ModelGauss2DRotX2 (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelGauss2DRotX2, true, C, false>;
  k.rk = pass_kernel<ModelGauss2DRotX2, false, C, false>;
  k.jkw = pass_kernel<ModelGauss2DRotX2, true, C, true>;
  k.rkw = pass_kernel<ModelGauss2DRotX2, false, C, true>;
  k.jkp = pass_kernel<ModelGauss2DRotX2, true, C, false, PassCfg<ModelGauss2DRotX2, true>::P, PassCfg<ModelGauss2DRotX2, true>::TPB, PassCfg<ModelGauss2DRotX2, true>::MINB, true>;
  k.jkpw = pass_kernel<ModelGauss2DRotX2, true, C, true, PassCfg<ModelGauss2DRotX2, true>::P, PassCfg<ModelGauss2DRotX2, true>::TPB, PassCfg<ModelGauss2DRotX2, true>::MINB, true>;
  k.jtpb = PassCfg<ModelGauss2DRotX2, true>::TPB;
  k.jptpb = PassCfg<ModelGauss2DRotX2, true>::TPB;
  k.jsplit = PassCfg<ModelGauss2DRotX2, true>::SPLIT;
  k.small = fit_small_kernel<ModelGauss2DRotX2, C, false>;
  k.smallw = fit_small_kernel<ModelGauss2DRotX2, C, true>;
  k.rtpb = PassCfg<ModelGauss2DRotX2, false>::TPB;
  return k;
}
Kernels kernels_gauss2d_x2(int coord) { return coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>(); }
}  // namespace jf

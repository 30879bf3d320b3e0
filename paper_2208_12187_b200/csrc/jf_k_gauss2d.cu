// jf_k_gauss2d.cu — pass-kernel instances for ModelGauss2DRot (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_pass.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelGauss2DRot, true, C, false>;
  k.rk = pass_kernel<ModelGauss2DRot, false, C, false>;
  k.jkw = pass_kernel<ModelGauss2DRot, true, C, true>;
  k.rkw = pass_kernel<ModelGauss2DRot, false, C, true>;
  k.jtpb = PassCfg<ModelGauss2DRot, true>::TPB;
  k.rtpb = PassCfg<ModelGauss2DRot, false>::TPB;
  return k;
}
Kernels kernels_gauss2d(int coord) { return coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>(); }
}  // namespace jf

// jf_k_gauss2d.cu — pass-kernel instances for ModelGauss2DRot (see jf_pass.cuh).
#include <cstdlib>

#include "jf_kernels.h"
#include "jf_moment.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelGauss2DRot, true, C, false>;
  k.rk = pass_kernel<ModelGauss2DRot, false, C, false>;
  k.jkw = pass_kernel<ModelGauss2DRot, true, C, true>;
  k.rkw = pass_kernel<ModelGauss2DRot, false, C, true>;
  k.jkp = pass_kernel<ModelGauss2DRot, true, C, false, PassCfg<ModelGauss2DRot, true>::P, PassCfg<ModelGauss2DRot, true>::TPB, PassCfg<ModelGauss2DRot, true>::MINB, true>;
  k.jkpw = pass_kernel<ModelGauss2DRot, true, C, true, PassCfg<ModelGauss2DRot, true>::P, PassCfg<ModelGauss2DRot, true>::TPB, PassCfg<ModelGauss2DRot, true>::MINB, true>;
  k.jtpb = PassCfg<ModelGauss2DRot, true>::TPB;
  k.jptpb = PassCfg<ModelGauss2DRot, true>::TPB;
  k.jsplit = PassCfg<ModelGauss2DRot, true>::SPLIT;
  k.small = fit_small_kernel<ModelGauss2DRot, C, false>;
  k.smallw = fit_small_kernel<ModelGauss2DRot, C, true>;
  k.rtpb = PassCfg<ModelGauss2DRot, false>::TPB;
  return k;
}
Kernels kernels_gauss2d(int coord) {
  Kernels k = coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>();
  // development aid: alternative launch shapes of the grid J-pass (JF_JVARIANT=1..3)
  if (coord == COORD_GRID) {
    // unweighted implicit grid: the moment-form J-pass (jf_moment.cuh)
    k.jk = moment_pass_kernel<16, 128, 3>;
    k.jtpb = 128;
    if (const char* v = getenv("JF_JVARIANT")) {
      const int var = atoi(v);
      if (var == 9) { k.jk = pass_kernel<ModelGauss2DRot, true, COORD_GRID, false>; k.jtpb = 256; }  // dual-number kernel
      if (var == 11) { k.jk = moment_pass_kernel<8, 128, 3>; }
      if (var == 12) { k.jk = moment_pass_kernel<8, 128, 4>; }
      if (var == 13) { k.jk = moment_pass_kernel<16, 128, 4>; }
      if (var == 14) { k.jk = moment_pass_kernel<8, 128, 5>; }
      if (var == 15) { k.jk = moment_pass_kernel<4, 128, 4>; }
      if (var == 16) { k.jk = moment_pass_kernel<16, 128, 3, 1>; }
      if (var == 17) { k.jk = moment_pass_kernel<16, 128, 3, 2>; }
      if (var == 18) { k.jk = moment_pass_kernel<16, 128, 3, 8>; }
      if (var == 19) { k.jk = moment_pass_kernel<8, 128, 3, 8>; }
    }
  }
  return k;
}
}  // namespace jf

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
template <int L, int TPB, int MINB, int SEEDN = 4, int STAGES = 0>
static void use_moment(Kernels& k) {
  auto f = moment_pass_kernel<L, TPB, MINB, SEEDN, STAGES>;
  k.jk = f;
  k.jtpb = TPB;
  k.jsmem = moment_zbuf_bytes(L, TPB, STAGES);
  if (k.jsmem > 0) cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, k.jsmem);
}

Kernels kernels_gauss2d(int coord) {
  Kernels k = coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>();
  if (coord == COORD_GRID) {
    // unweighted implicit grid: the moment-form J-pass (jf_moment.cuh)
    use_moment<16, 128, 3>(k);
    if (const char* v = getenv("JF_JVARIANT")) {  // development aid: alternative shapes
      const int var = atoi(v);
      if (var == 9) { k.jk = pass_kernel<ModelGauss2DRot, true, COORD_GRID, false>; k.jtpb = 256; k.jsmem = 0; }  // dual numbers
      if (var == 11) use_moment<8, 128, 3>(k);
      if (var == 12) use_moment<8, 128, 4>(k);
      if (var == 13) use_moment<16, 128, 3, 8>(k);
      if (var == 20) use_moment<16, 128, 3, 4, 2>(k);
      if (var == 21) use_moment<16, 128, 3, 4, 3>(k);
      if (var == 22) use_moment<8, 128, 4, 4, 2>(k);
      if (var == 23) use_moment<8, 128, 4, 4, 3>(k);
      if (var == 24) use_moment<16, 128, 4, 4, 2>(k);
      if (var == 25) use_moment<8, 128, 5, 4, 2>(k);
    }
  }
  return k;
}
}  // namespace jf

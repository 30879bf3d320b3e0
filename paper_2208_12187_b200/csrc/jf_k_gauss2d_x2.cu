// jf_k_gauss2d_x2.cu — pass-kernel instances for ModelGauss2DRotX2 (see jf_pass.cuh).
#include "jf_kernels.h"
#include <cstdlib>

#include "jf_moment2.cuh"

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
template <int L, int TC, int NW, bool ROLLED = false>
static void use_moment2(Kernels& k) {
  if (k.jwtpb == 0) {  // the dual-number kernel stays in use for weighted passes
    k.jwtpb = k.jtpb;
    k.jwsplit = k.jsplit ? 1 : 0;
  }
  k.jk = moment2_task_kernel<L, TC, NW, ROLLED>;
  k.jtpb = NW * 32;
  k.jsmem = moment2_task_smem_bytes(NW);
  k.jsplit = false;
}
void kernel_attrs_init_x2() {
  cudaFuncSetAttribute((const void*)moment2_task_kernel<8, 8, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment2_task_smem_bytes(12));
  cudaFuncSetAttribute((const void*)moment2_task_kernel<8, 8, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment2_task_smem_bytes(8));
  cudaFuncSetAttribute((const void*)moment2_task_kernel<8, 4, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment2_task_smem_bytes(12));
  cudaFuncSetAttribute((const void*)moment2_task_kernel<8, 8, 12, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment2_task_smem_bytes(12));
  cudaFuncSetAttribute((const void*)moment2_task_kernel<16, 4, 12, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment2_task_smem_bytes(12));
}
Kernels kernels_gauss2d_x2(int coord) {
  Kernels k = coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>();
  if (coord == COORD_GRID) {
    // unweighted implicit grid: the moment-form J-pass (jf_moment2.cuh)
    const char* v = getenv("JF_X2VARIANT");  // development aid: 9 = the dual-number kernel
    const int var = v ? atoi(v) : 0;
    if (var == 1) use_moment2<8, 8, 8>(k);
    else if (var == 2) use_moment2<8, 4, 12>(k);
    else if (var == 4) use_moment2<16, 4, 12, true>(k);
    else if (var == 5) use_moment2<8, 8, 12>(k);  // unrolled fast path
    else if (var != 9) use_moment2<8, 8, 12, true>(k);
  }
  return k;
}
}  // namespace jf

// jf_k_gauss2d.cu — pass-kernel instances for ModelGauss2DRot (see jf_pass.cuh).
#include <cstdlib>

#include "jf_kernels.h"
#include "jf_moment.cuh"
#include "jf_moment_stream.cuh"

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
template <int L, int TPB, int MINB, int SEEDN = 4, int STG = 0>
static void use_moment(Kernels& k) {
  if (k.jwtpb == 0) {  // the dual-number kernel stays in use for weighted passes
    k.jwtpb = k.jtpb;
    k.jwsplit = k.jsplit ? 1 : 0;
  }
  auto f = moment_pass_kernel<L, TPB, MINB, SEEDN, STG>;
  k.jk = f;
  k.jtpb = TPB;
  k.jsmem = moment_smem_bytes(L, TPB, STG);
}

template <int L, int TC, int NW, int SEEDN = 4, int DBGZ = 0, int FASTP = 1>
static void use_task(Kernels& k) {
  if (k.jwtpb == 0) {  // the dual-number kernel stays in use for weighted passes
    k.jwtpb = k.jtpb;
    k.jwsplit = k.jsplit ? 1 : 0;
  }
  k.jk = moment_task_kernel<L, TC, NW, SEEDN, DBGZ, FASTP>;
  k.jtpb = NW * 32;
  k.jsmem = moment_task_smem_bytes(NW);
}
template <int L, int TC, int NW, int SEEDN = 4, int DBGZ = 0, int FASTP = 1>
static void attr_task() {
  cudaFuncSetAttribute((const void*)moment_task_kernel<L, TC, NW, SEEDN, DBGZ, FASTP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment_task_smem_bytes(NW));
}
template <int L, int TPB, int MINB, int SEEDN, int STG>
static void attr_moment() {
  cudaFuncSetAttribute((const void*)moment_pass_kernel<L, TPB, MINB, SEEDN, STG>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, moment_smem_bytes(L, TPB, STG));
}
template <int L, int NW, int SEEDN>
static void use_stream(Kernels& k) {
  if (k.jwtpb == 0) {  // the dual-number kernel stays in use for weighted passes
    k.jwtpb = k.jtpb;
    k.jwsplit = k.jsplit ? 1 : 0;
  }
  k.jk = moment_stream_kernel<L, NW, SEEDN>;
  k.jtpb = NW * 32;
  k.jsmem = moment_stream_smem_bytes(NW);
}
template <int L, int NW, int SEEDN>
static void attr_stream() {
  cudaFuncSetAttribute((const void*)moment_stream_kernel<L, NW, SEEDN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment_stream_smem_bytes(NW));
}
void kernel_attrs_init() {
  attr_stream<16, 12, 8>();
  attr_stream<16, 16, 8>();
  attr_stream<8, 16, 8>();
  attr_task<16, 4, 12, 4, 0, 2>();
  attr_task<16, 2, 12>();
  attr_task<16, 4, 16>();
  attr_task<16, 8, 12>();
  attr_task<8, 8, 16>();
  attr_task<32, 2, 8, 2>();
  attr_task<16, 4, 12, 4, 1>();
  attr_task<16, 4, 12, 4, 0, 0>();
  attr_task<16, 4, 12, 4, 0, 1>();
  attr_task<16, 4, 12, 4, 0, 2>();
  attr_moment<16, 128, 3, 4, 3>();
  attr_moment<16, 128, 3, 4, 4>();
  attr_moment<8, 128, 4, 8, 4>();
  attr_moment<8, 128, 4, 8, 6>();
  attr_moment<16, 256, 1, 4, 3>();
  attr_moment<32, 128, 2, 2, 3>();
  attr_moment<16, 128, 2, 4, 6>();
}

Kernels kernels_gauss2d(int coord) {
  Kernels k = coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>();
  if (coord == COORD_GRID) {
    // unweighted implicit grid: the moment-form J-pass (jf_moment.cuh),
    // task-scheduled, one block of 12 warps per SM
    use_stream<16, 12, 8>(k);
    if (const char* v = getenv("JF_JVARIANT")) {  // development aid: alternative shapes
      const int var = atoi(v);
      if (var == 50) use_task<16, 4, 12, 4, 0, 2>(k);  // r1 task-scheduled kernel
      if (var == 51) use_stream<16, 16, 8>(k);
      if (var == 52) use_stream<8, 16, 8>(k);
      if (var == 9) { k.jk = pass_kernel<ModelGauss2DRot, true, COORD_GRID, false>; k.jtpb = 256; k.jsmem = 0; }  // dual numbers
      if (var == 1) use_moment<16, 128, 3>(k);  // static per-warp split (r1d)
      if (var == 11) use_moment<8, 128, 4>(k);
      if (var == 30) use_task<16, 4, 12>(k);
      if (var == 31) use_task<16, 2, 12>(k);
      if (var == 32) use_task<16, 4, 16>(k);
      if (var == 33) use_task<16, 8, 12>(k);
      if (var == 34) use_task<8, 8, 16>(k);
      if (var == 35) use_task<32, 2, 8, 2>(k);
      if (var == 39) use_task<16, 4, 12, 4, 1>(k);  // compute-only probe (wrong results)
      if (var == 40) use_task<16, 4, 12, 4, 0, 0>(k);  // no whole-task fast path
      if (var == 42) use_task<16, 4, 12, 4, 0, 1>(k);  // unrolled whole-task fast path (r1i)
      if (var == 13) use_moment<32, 128, 2, 2>(k);
      if (var == 20) use_moment<16, 128, 3, 4, 3>(k);
      if (var == 21) use_moment<16, 128, 3, 4, 4>(k);
      if (var == 22) use_moment<8, 128, 4, 8, 4>(k);
      if (var == 23) use_moment<8, 128, 4, 8, 6>(k);
      if (var == 24) use_moment<16, 256, 1, 4, 3>(k);
      if (var == 25) use_moment<32, 128, 2, 2, 3>(k);
      if (var == 26) use_moment<16, 128, 2, 4, 6>(k);
    }
  }
  return k;
}
}  // namespace jf

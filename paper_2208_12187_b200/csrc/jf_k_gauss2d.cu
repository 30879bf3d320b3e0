// jf_k_gauss2d.cu — pass-kernel instances for ModelGauss2DRot (see jf_pass.cuh).
#include "jf_kernels.h"
#include "jf_moment_stream.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelGauss2DRot, true, C, false>;
  k.rk = pass_kernel<ModelGauss2DRot, false, C, false>;
  k.jkw = pass_kernel<ModelGauss2DRot, true, C, true>;
  k.rkw = pass_kernel<ModelGauss2DRot, false, C, true>;
  k.jtpb = PassCfg<ModelGauss2DRot, true>::TPB;
  k.jsplit = PassCfg<ModelGauss2DRot, true>::SPLIT;
  k.small = fit_small_kernel<ModelGauss2DRot, C, false>;
  k.batch = fit_batch_kernel<ModelGauss2DRot, C, false>;
  k.batchw = fit_batch_kernel<ModelGauss2DRot, C, true>;
  k.smallw = fit_small_kernel<ModelGauss2DRot, C, true>;
  k.rtpb = PassCfg<ModelGauss2DRot, false>::TPB;
  return k;
}

// The moment-form J-pass (R34): L = 16 points per lane per warp-chunk, 12
// warps per block (one block per SM), recurrence re-seeded every 8 chunks,
// z staged by bulk copies (TMA) through a 3-chunk ring per warp.
constexpr int JL = 16, JNW = 12, JSEED = 8, JSTG = 3;
#define JSTREAM moment_stream_kernel<JL, JNW, JSEED, JSTG>

void kernel_attrs_init() {
  cudaFuncSetAttribute((const void*)JSTREAM, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment_stream_smem_bytes(JNW, JL, JSTG));

}

Kernels kernels_gauss2d(int coord) {
  Kernels k = coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>();
  if (coord == COORD_GRID) {
    // unweighted implicit grid: the moment-form J-pass; weighted passes keep
    // the dual-number kernel and its launch shape
    k.jwtpb = k.jtpb;
    k.jwsplit = k.jsplit ? 1 : 0;
    k.jk = JSTREAM;
    k.jtpb = JNW * 32;
    k.jsmem = moment_stream_smem_bytes(JNW, JL, JSTG);
    static_assert(moment_stream_smem_bytes(JNW, JL, JSTG) >= (int)fused_solver_smem_bytes(), "solver scratch");
    k.jfused = true;

  }
  return k;
}
}  // namespace jf

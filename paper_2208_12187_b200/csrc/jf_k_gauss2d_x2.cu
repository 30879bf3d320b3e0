// jf_k_gauss2d_x2.cu — pass-kernel instances for ModelGauss2DRotX2 (see jf_pass.cuh).
#include "jf_kernels.h"

#include "jf_moment2.cuh"

namespace jf {
template <int C>
static Kernels make() {
  Kernels k;
  k.jk = pass_kernel<ModelGauss2DRotX2, true, C, false>;
  k.rk = pass_kernel<ModelGauss2DRotX2, false, C, false>;
  k.jkw = pass_kernel<ModelGauss2DRotX2, true, C, true>;
  k.rkw = pass_kernel<ModelGauss2DRotX2, false, C, true>;
  k.jtpb = PassCfg<ModelGauss2DRotX2, true>::TPB;
  k.jsplit = PassCfg<ModelGauss2DRotX2, true>::SPLIT;
  k.small = fit_small_kernel<ModelGauss2DRotX2, C, false>;
  k.batch = fit_batch_kernel<ModelGauss2DRotX2, C, false>;
  k.batchw = fit_batch_kernel<ModelGauss2DRotX2, C, true>;
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
  // (the moment kernel itself runs on any grid, but its fallback to the
  // dual-number body — narrow or elongated peaks — splits the n = 13 triangle
  // across two halves of the grid: at least two blocks)
  k.jsplit = true;
  static_assert(moment2_task_smem_bytes(12) >= (int)fused_solver_smem_bytes(), "solver scratch");
  k.jfused = true;  // speculative one-GPU fits: the solver step in the pass's last block
}
void kernel_attrs_init_x2() {
  cudaFuncSetAttribute((const void*)moment2_task_kernel<8, 8, 12, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       moment2_task_smem_bytes(12));
}
Kernels kernels_gauss2d_x2(int coord) {
  Kernels k = coord == COORD_EXPLICIT ? make<COORD_EXPLICIT>() : make<COORD_GRID>();
  if (coord == COORD_GRID) {
    // unweighted implicit grid: the moment-form J-pass (jf_moment2.cuh, R35),
    // task sub-runs as a rolled loop
    use_moment2<8, 8, 12, true>(k);
  }
  return k;
}
}  // namespace jf

// jf_kernels.h — host-side handles of the pass-kernel instances, one
// translation unit per model (jf_k_*.cu) so they compile in parallel.
#pragma once

#include "jf_common.cuh"

namespace jf {
struct FitState;
// Pass kernels: (device args or nullptr, fit state, WHILE handle, use it, args by value).
// A fit graph passes the context's device-resident PassArgs (so one cached
// graph serves any data); a plain pass passes nullptr and its args by value
// (immutable once enqueued or captured).
using KernelFn = void (*)(const PassArgs*, FitState*, cudaGraphConditionalHandle, int, const PassArgs);
using SmallFitFn = void (*)(const PassArgs*, FitState*);
using BatchFn = void (*)(const BatchArgs);
struct Kernels {
  KernelFn jk = nullptr;   // J-pass (value + Jacobian + fused Gram); in a fit also the TSQR second pass
  KernelFn rk = nullptr;   // residual-only pass
  KernelFn jkw = nullptr;  // weighted variants (App. C)
  KernelFn rkw = nullptr;
  int jtpb = 256, rtpb = 256;  // threads per block of the J / r kernels
  int jsmem = 0;               // dynamic shared memory of the J kernel (bytes)
  bool jfused = false;         // jk runs the solver step in its last block (PassArgs::fused)
  bool jsplit = false;         // J grid split in two halves (even grid >= 2)
  int jwtpb = 0;               // weighted J kernel's block size / split when jk is a moment kernel
  int jwsplit = -1;            //   (0 / -1: same as jtpb / jsplit)
  SmallFitFn small = nullptr;  // whole-fit single-block kernel (small m), unweighted / weighted
  SmallFitFn smallw = nullptr;
  BatchFn batch = nullptr;     // many small fits per launch (one warp per fit), unweighted / weighted
  BatchFn batchw = nullptr;
};
Kernels kernels_linear(int coord);
Kernels kernels_exp_decay(int coord);
Kernels kernels_gauss1d(int coord);
Kernels kernels_gauss2d(int coord);
Kernels kernels_gauss2d_x2(int coord);
// Per-device function attributes (opt-in dynamic shared memory), set once per
// device when its first context is created — never during a pass, when an
// attribute call could wait on the spinning kernels of emulated peer ranks.
void kernel_attrs_init();
void kernel_attrs_init_x2();
}  // namespace jf

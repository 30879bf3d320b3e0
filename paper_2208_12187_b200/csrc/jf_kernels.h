// jf_kernels.h — host-side handles of the pass-kernel instances, one
// translation unit per model (jf_k_*.cu) so they compile in parallel.
#pragma once

#include "jf_common.cuh"

namespace jf {
struct FitState;
using KernelFn = void (*)(const PassArgs*, FitState*, cudaGraphConditionalHandle, int);
using SmallFitFn = void (*)(const PassArgs*, FitState*);
struct Kernels {
  KernelFn jk = nullptr;   // J-pass (value + dual Jacobian + fused Gram)
  KernelFn rk = nullptr;   // residual-only pass
  KernelFn jkw = nullptr;  // weighted variants (App. C)
  KernelFn rkw = nullptr;
  KernelFn jkp = nullptr;   // J-pass with the TSQR preconditioner (CholeskyQR2 second pass)
  KernelFn jkpw = nullptr;
  int jtpb = 256, rtpb = 256;  // threads per block of the J / r kernels
  int jptpb = 256;             // threads per block of the preconditioned J kernel
  int jsmem = 0;               // dynamic shared memory of the J kernel (bytes)
  bool jsplit = false;         // J grid split in two halves (even grid >= 2)
  int jwtpb = 0;               // weighted J kernel's block size / split when jk is a moment kernel
  int jwsplit = -1;            //   (0 / -1: same as jtpb / jsplit)
  SmallFitFn small = nullptr;  // whole-fit single-block kernel (small m), unweighted / weighted
  SmallFitFn smallw = nullptr;
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

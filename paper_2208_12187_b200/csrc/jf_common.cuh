// jf_common.cuh — shared device-side definitions of the B200 hot path.
#pragma once

#include <cstdio>

#include <cstdint>
#include <cuda_runtime.h>

namespace jf {

constexpr int NMAX = 16;                               // JF_MAX_N
constexpr int KMAX = (NMAX + 1) * (NMAX + 2) / 2 + 1;  // K-vector length for n = 16
constexpr int BLOCK = 256;                             // threads per pass block
constexpr int NWARP = BLOCK / 32;
constexpr unsigned FULL = 0xffffffffu;

// Checked builds (JF_CHECKED=1 python -m paper_2208_12187_b200.build; never
// shipped): device-side bounds checks on every global read of the data and on
// the bulk-copy ranges; a failed check prints where and traps the kernel.
// The substitute for compute-sanitizer, which the GPU pool does not allow.
#ifndef JF_CHECKED
#define JF_CHECKED 0
#endif
#define JF_DCHECK(cond)                                                                                  \
  do {                                                                                                   \
    if (JF_CHECKED && !(cond)) {                                                                         \
      printf("JF_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,          \
             (int)blockIdx.x, (int)threadIdx.x);                                                         \
      __trap();                                                                                          \
    }                                                                                                    \
  } while (0)

// K-vector slot of W^T W entry (j, k), j <= k <= n, W = [J | r] (jf.h).
__host__ __device__ constexpr int tri_slot(int n, int j, int k) {
  return j * (n + 1) - (j * (j - 1)) / 2 + (k - j);
}
__host__ __device__ constexpr int tri_count(int n) { return (n + 1) * (n + 2) / 2; }

enum CoordMode : int32_t {
  COORD_EXPLICIT = 0,  // y arrays: t[m] (d=1) or X[m], Y[m] (d=2)
  COORD_GRID = 1,      // implicit pixel grid (W, row0): X = i % W, Y = i / W + row0
  COORD_IMPLICIT_T = 2 // t_i = t0 + (index0 + i) dt
};

// Epilogue run by the last block of a pass kernel after the deterministic combine.
enum Epilogue : int32_t { EPI_NONE = 0, EPI_FIT = 1 };

// Multi-GPU mailbox (see jf_comm.cu).  mbox[p] is rank p's mailbox as mapped
// in this process (mbox[rank] is local).  Layout of one mailbox:
//   double slot[2][nranks][KMAX]  (parity-double-buffered by epoch)
//   uint64 flag[nranks]           (epoch written by each sender after its data)
struct CommDev {
  int32_t rank, nranks;
  double* mbox_data[8];
  unsigned long long* mbox_flag[8];
  unsigned long long epoch;  // host-side base; the device uses st->comm_epoch
  unsigned long long timeout_ns;  // a peer that does not arrive within this is reported (JF_ECOMM)
};

// Kernel inputs that stay fixed during one call (device-resident, so a cached
// CUDA graph can be replayed for any data).
struct PassArgs {
  const double* z;      // observations [m]
  const double* y0;     // t[m] or X[m] (COORD_EXPLICIT)
  const double* y1;     // Y[m] (COORD_EXPLICIT, d=2)
  const double* wsig;   // 1/sigma_i [m] or nullptr (App. C, Eq. C13-C16)
  int64_t m;            // points in this shard
  int64_t W;            // grid width (COORD_GRID)
  int64_t row0;         // first row of this shard (COORD_GRID)
  int64_t index0;       // first global index (COORD_IMPLICIT_T)
  double t0, dt;        // COORD_IMPLICIT_T
  int32_t coord;        // CoordMode
  int32_t epilogue;     // Epilogue
  const double* x;      // parameters to evaluate at (device, n doubles) for EPI_NONE
  double* partials;     // [gridDim.x][KS] per-block partial K-vectors
  unsigned int* ticket; // last-block ticket (reset by the last block)
  double* out;          // combined K-vector (EPI_NONE)
  int* err;             // EPI_NONE: set to JF_ECOMM (-5) if the cross-rank combine failed
  const double* precond; // EPI_NONE TSQR second pass: P = R1^-1, (n+1)^2 row-major upper triangular
  int32_t use_comm;     // 1: combine across ranks through the mailboxes
  int32_t no_chain;     // debug (JF_DEBUG_NOCHAIN): return the Gram in the alt coordinates (a, 2b, c2)
  unsigned long long* dbg; // debug (JF_DEBUG_STAMPS): per-warp [smid, t_start, t_loop_end, t_exit] (moment kernel)
  // the parameter-only prologue of the n = 7 moment J-pass, precomputed for
  // x by the caller (host x) — n = 7: {A, x0, y0, a, 2b, c2, off, rho}; n = 13:
  // {A, x0, y0, a, 2b, c2} of each component, off, rho1, rho2; has_pre = 0: in-kernel
  double pre[16];
  int32_t has_pre;
  int32_t fused;        // fit of the n = 7 moment J-pass: the solver step runs in the pass's last block
                        // (its dynamic shared memory as scratch) — no solver kernel between passes
  CommDev comm;
};

// Batched many-small-fits (jf_curve_fit_batch): one warp
// per fit, the whole TRF of a fit inside one persistent kernel.
struct BatchResult {  // = jf_batch_result (include/jf.h)
  double x[NMAX];
  double cost, optimality;
  int32_t status, nfev, njev, nit;
};
struct QRState;
struct FitState;
struct BatchArgs {
  PassArgs base;            // the arguments of fit 0 (z, y0, y1, wsig at their base pointers)
  int64_t nfits;
  int64_t z_stride;         // doubles between consecutive fits' z (and sigma)
  int64_t y_stride;         // doubles between consecutive fits' coordinates (0: shared)
  const double* p0;         // nfits x n, or nullptr: curve_fit's default p0 for every fit
  const FitState* tmpl;     // configuration shared by every fit (bounds, tolerances, solver mode)
  QRState* qr;              // one TSQR working set per block
  BatchResult* out;         // nfits results
};

}  // namespace jf

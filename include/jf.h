/*
 * jf.h — C ABI of the B200-native JAXFit hot path (libjfb200.so).
 *
 * What this library computes (citations are to /root/reference/PAPER.md,
 * "P:<line> §/Eq./Alg.", and to the build's readings in DESIGN.md §3 "R<k>"):
 *
 *   minimise f(x) = 1/2 * sum_i r_i(x)^2,  r_i(x) = h(y_i; x) - z_i      (Eq. 1-2)
 *
 * by the trust-region-reflective method of P:40-212 §II (Alg. 1-3,
 * Eq. 3-15), with the SVD solve of P:314-343 App. B, unconstrained or with
 * box bounds lb <= x <= ub (Coleman-Li reflective scaling, "SciPy's
 * adapted version"; reading R19).  h is one of a fixed set of built-in models
 * (jf_model).  Every per-iteration pass over the m data points runs in
 * hand-written sm_100a CUDA kernels and reduces, in fp64, to
 *     cost = 1/2 r^T r (Eq. 2),  g = J^T r (Eq. 4),  G = J^T J (Eq. 5, Gauss-Newton B),
 * never materialising J.  The Jacobian is forward-mode: by dual
 * numbers carrying the whole row for the 1-D models, explicit coordinates and
 * weighted fits; for the rotated 2-D Gaussians on an implicit pixel grid
 * (unweighted) by the moment form (readings R33-R35): the same
 * partials regrouped as fixed linear combinations of per-pass moments of
 * exp(-q) along image rows, mapped to (cost, g, G) once per pass.  The n x n trust-region subproblem (Eq. 9-14,
 * Alg. 2) runs in a single-warp device kernel; the iteration (Alg. 1, 3) is a
 * device state machine driven by a CUDA graph with a conditional WHILE node.
 *
 * Conventions shared by every entry point
 * ----------------------------------------
 *  - All floating point is IEEE fp64.  All integers are fixed width.
 *  - All pointers are caller-owned.  Host inputs are copied; device inputs
 *    (opts->inputs_on_device != 0) are read in place during the call only.
 *    The library keeps no caller pointer after a call returns.
 *  - Return value >= 0: success (jf_curve_fit: the solver status below).
 *    Return value < 0: one of the JF_E* error codes; nothing else escapes
 *    the ABI (no C++ exceptions, no abort).  jf_strerror() names the code.
 *  - Calls on one device serialise on an internal per-device mutex; calls on
 *    different devices may run concurrently.
 *  - Data layout ("y"): for 1-D models (jf_model_ydim == 1) y is t[m].  For
 *    2-D models y is the SoA pair X[m] followed by Y[m] (2*m doubles), or
 *    y == NULL with an implicit pixel grid (opts->grid_w, grid_h, grid_row0):
 *    point i is pixel (row = i / grid_w, col = i % grid_w), X = col,
 *    Y = row + grid_row0 (reading R21: pixel centres at integer coordinates).
 *    For 1-D models y == NULL means t_i = opts->t0 + (opts->index0 + i)*opts->dt.
 *  - The per-pass reduction vector ("K-vector", fp64, K = (n+1)(n+2)/2 + 1):
 *    the upper triangle, row-major, of W^T W with W = [J | r] (m x (n+1)),
 *    slot(j,k) = j*(n+1) - j*(j-1)/2 + (k-j) for 0 <= j <= k <= n, followed
 *    by one slot holding the count of non-finite residuals (reading R17).
 *    So G_jk = slot(j,k) (j,k < n), g_j = slot(j,n), r^T r = slot(n,n).
 *
 * Ownership, threading and error behaviour are restated per function below.
 */
#ifndef JF_H_
#define JF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JF_MAX_N 16              /* largest parameter count the kernels support */
#define JF_COMM_HANDLE_BYTES 256 /* size of one rank's exported mailbox handle */

/* Built-in models h(y; x).  Parameter order is fixed (reading R21):
 *  JF_LINEAR         n=2  d=1  x0*t + x1                         (closed-form pin)
 *  JF_EXP_DECAY      n=3  d=1  a*exp(-b*t) + c, x=(a,b,c)
 *  JF_GAUSS1D        n=4  d=1  A*exp(-(t-mu)^2/(2 s^2)) + c, x=(A,mu,s,c)
 *  JF_GAUSS2D_ROT    n=7  d=2  A*exp(-(a dx^2 + 2b dx dy + c2 dy^2)) + off,
 *                    x=(A,x0,y0,sx,sy,theta,off), dx=X-x0, dy=Y-y0,
 *                    a=cos^2/(2sx^2)+sin^2/(2sy^2), b=sin2t*(1/(4sy^2)-1/(4sx^2)),
 *                    c2=sin^2/(2sx^2)+cos^2/(2sy^2)   (§IV "2D rotated, elliptical
 *                    Gaussians ... seven fitting parameters"; form from SPEC.md S:463)
 *  JF_GAUSS2D_ROT_X2 n=13 d=2  two JF_GAUSS2D_ROT without offsets plus one shared offset,
 *                    x=(A1,x1,y1,sx1,sy1,t1, A2,x2,y2,sx2,sy2,t2, off)                  */
typedef enum {
  JF_LINEAR = 0,
  JF_EXP_DECAY = 1,
  JF_GAUSS1D = 2,
  JF_GAUSS2D_ROT = 3,
  JF_GAUSS2D_ROT_X2 = 4
} jf_model;

/* Diagonal scaling D of P:94-100 Eq. 7 (reading R3).
 *  JAC:   D_k = diag(max_{j<=k} ||J_{:,i}(x_j)||), zero column -> 1 at k=0
 *  ONES:  D = I
 *  ARRAY: D = diag(1 / x_scale), x_scale given by the caller (n finite > 0) */
typedef enum { JF_XSCALE_JAC = 0, JF_XSCALE_ONES = 1, JF_XSCALE_ARRAY = 2 } jf_xscale;

/* How the per-pass reduction feeds App. B's SVD:
 *  GRAM: fp64 Gram G = J^T J; Cholesky Gauss-Newton trial, eigendecomposition
 *        of the scaled Gram when Alg. 2 needs alpha > 0
 *  TSQR: R factor of W = [J | r] by CholeskyQR2 (a Gram pass, then a pass
 *        accumulating (W R1^-1)^T (W R1^-1); R = chol(.) R1) while its
 *        certificate bounds cond(W)^2 by 1e14, else by shifted CholeskyQR3
 *        (R1 = chol(W^T W + s I), then CholeskyQR2 on W R1^-1: one pass
 *        more; cond(W) up to ~1e16); SVD of the scaled R by one-sided Jacobi
 *        (two or three passes per accepted step)
 *  AUTO: TSQR if cond(J D^-1)^2 estimated at x0 — or at an accepted step —
 *        exceeds 1e6, else GRAM (the default) */
typedef enum { JF_SOLVE_AUTO = 0, JF_SOLVE_GRAM = 1, JF_SOLVE_TSQR = 2 } jf_solver;

/* Which pass evaluates a trial point x + w (Eq. 15 needs f(x+w)):
 *  SPECULATIVE:  the full J-pass at every trial, so an accepted step already has
 *                J(x+w) (one pass per trial; identical iterates and counts)
 *  CONSERVATIVE: a residual-only pass per trial, plus a J-pass on acceptance   */
typedef enum { JF_POLICY_SPECULATIVE = 0, JF_POLICY_CONSERVATIVE = 1 } jf_policy;

/* Solver status (>= 0), SciPy's codes (reading R16):
 *  0 max_nfev reached, 1 gtol, 2 ftol, 3 xtol, 4 ftol and xtol. */
enum {
  JF_OK = 0,
  JF_EINVAL = -1,       /* null pointer, m < 1, n != jf_model_nparams(model), lb >= ub,
                           NaN bound, bad x_scale, y == NULL without grid, grid_w*grid_h != m */
  JF_EINFEASIBLE = -2,  /* p0 outside [lb, ub] (reading R18) */
  JF_ENONFINITE = -3,   /* residuals at p0 not all finite (reading R18) */
  JF_ECUDA = -4,        /* a CUDA runtime call failed (no device, launch failure, ...) */
  JF_ECOMM = -5,        /* multi-GPU combine failed (bad handles, peer timeout) */
  JF_ENOMEM = -6        /* device or pinned host allocation failed */
};

typedef struct jf_comm jf_comm;

typedef struct jf_opts {
  double ftol, xtol, gtol;      /* termination tolerances, default 1e-8 each (R16)            */
  int32_t max_nfev;             /* 0 -> 100*n (R16)                                            */
  int32_t x_scale_mode;         /* jf_xscale, default JF_XSCALE_JAC                           */
  const double* x_scale;        /* host, n entries, used iff x_scale_mode == JF_XSCALE_ARRAY  */
  int32_t solver;               /* jf_solver, default JF_SOLVE_AUTO (jf_pass: always the Gram) */
  int32_t policy;               /* jf_policy, default JF_POLICY_SPECULATIVE                   */
  int64_t grid_w, grid_h;       /* implicit pixel grid for 2-D models when y == NULL          */
  int64_t grid_row0;            /* global row of this shard's first row (sharded images)      */
  double t0, dt;                /* implicit t for 1-D models when y == NULL                   */
  int64_t index0;               /* global index of this shard's first point (1-D, implicit t) */
  const double* sigma;          /* optional per-point sigma_i > 0 (P:346-352 Eq. C1, C13-C16):
                                   r~_i = r_i / sigma_i, J~ rows / sigma_i.  Same residency as z */
  int32_t device;               /* CUDA device ordinal, default 0                             */
  int32_t inputs_on_device;     /* 0: y, z, sigma are host pointers; 1: device pointers       */
  void* stream;                 /* cudaStream_t to run on, NULL -> library's own stream       */
  jf_comm* comm;                /* NULL: one GPU; else y, z, m are this rank's shard          */
  int32_t use_graph;            /* 1 (default): CUDA graph with conditional WHILE node;
                                   0: host-driven loop (one kernel launch + flag read per trial) */
  int32_t trace_cap;            /* > 0: record up to trace_cap trials into trace[]             */
  double* trace;                /* host, trace_cap * JF_TRACE_FIELDS doubles, caller-owned     */
  int64_t m_global;             /* sharded fits: total m over ranks (0 -> summed over the ranks
                                   by one combine through the comm at the start of the fit)      */
  int64_t capacity;             /* > 0: size every pass and the fit's CUDA graph for `capacity`
                                   points (>= m).  One cached graph then serves every m <=
                                   capacity; m itself is read from device memory at run time
                                   and points i >= m are never read (the masking of P:283-311
                                   App. A without dummy data; reading R26).  0: sized for m   */
  int32_t flags;                /* JF_FLAG_*, default 0                                         */
  int32_t pad_opts_;
  const double* x_host;         /* jf_pass_device: optional host copy of x_dev's n values, read at
                                   the call.  The rotated 2D Gaussian's moment J-pass then takes its
                                   parameter-only prologue (the quadratic form's a, 2b, c2 from
                                   sx, sy, theta; R34) precomputed by the call instead of computing
                                   it in every thread — as inside jf_curve_fit, where the solver
                                   kernel computes it.  NULL (default): computed in the kernel.
                                   Must equal x_dev's contents; other calls ignore it.          */
} jf_opts;

/* jf_opts.flags */
#define JF_FLAG_BATCH_SHARED_Y 2  /* jf_curve_fit_batch: y holds ONE set of coordinates for all fits */
#define JF_FLAG_ALT_COORDS 1  /* passes of the rotated Gaussians return W^T W in the alternative
                                 coordinates (a, 2b, c2) of their quadratic form — the first
                                 stage of the two-stage chain rule (reading R33) — for tests */

/* One trace record per trial (Alg. 1-3 quantities), in this order:
 *  nit, nfev, njev, cost, cost_new, Delta, alpha, ratio, ||p_h||, ||step||, pred, branch
 *  (branch of the Coleman-Li step selection: 0 interior, 1 reflected, 2 truncated,
 *   3 scaled gradient; -1 unconstrained) */
#define JF_TRACE_FIELDS 12

typedef struct jf_result {
  double x[JF_MAX_N];           /* final iterate                                               */
  double cost;                  /* 1/2 ||r(x)||^2 at x (Eq. 2)                                 */
  double optimality;            /* ||g||_inf (bounded: ||g * v||_inf) at x                     */
  double grad[JF_MAX_N];        /* g = J^T r at x (Eq. 4)                                      */
  double gram[JF_MAX_N * JF_MAX_N]; /* G = J^T J at x, n*n row-major (Eq. 5)                   */
  double pcov[JF_MAX_N * JF_MAX_N]; /* parameter covariance (curve_fit's pcov): pinv(G) *
                                   2 cost/(m-n), singular values below eps*max(m,n)*s_max dropped */
  int32_t status, nfev, njev, nit;
  int32_t n, trace_len;
  int8_t active_mask[JF_MAX_N]; /* -1 lower, +1 upper, 0 free (bounded fits; R19)              */
  int32_t kernel_launches;      /* device kernels this call launched                          */
  int32_t graph_reused;         /* 1: the fit replayed an already-instantiated CUDA graph      */
  double t_upload_s, t_solve_s; /* host wall time of the H2D copies and of the solve           */
  double t_epilogue_s;          /* device time in the single-warp solver epilogues (globaltimer) */
  double epilogue_cycles[8];    /* SM cycles in: eigensolver, trial solve, Coleman-Li step
                                   selection, whole solver step (diagnostics)                    */
  int32_t timeline_len, pad2_;
  double timeline_ns[64];       /* device timeline of the fit (ns from the first event): pass
                                   kernel start, pass end (last block), solver start, solver end */
} jf_result;

/* Fill *opts with the defaults above.  opts must be non-NULL. */
void jf_opts_default(jf_opts* opts);

/* n (number of parameters) of a model, or -1 for an unknown model. */
int32_t jf_model_nparams(int32_t model);

/* d (independent-variable dimension: 1 or 2) of a model, or -1. */
int32_t jf_model_ydim(int32_t model);

/* Length K of the per-pass reduction vector for a model, (n+1)(n+2)/2 + 1, or -1. */
int32_t jf_model_kslots(int32_t model);

/* jf_curve_fit — the whole fit (Alg. 1-3, App. B; bounded: R19).
 *  model, y, z, m: the data {y_i, z_i}, i < m.  z: m doubles.
 *  p0: n doubles initial guess (NULL: all ones, or for a bounded fit the
 *      midpoint of finite bounds / bound + 1 / bound - 1 / 1 as in curve_fit).
 *  lb, ub: n doubles each or NULL (= -inf / +inf); entries may be +-INFINITY.
 *      The bounded (Coleman-Li) path is used iff any bound is finite.
 *  opts: NULL means jf_opts_default().  out: caller-allocated, always written
 *      (out->status mirrors a negative return).
 * Returns the solver status (0..4) or a JF_E* error.  Blocks until done.   */
int32_t jf_curve_fit(int32_t model, const double* y, const double* z, int64_t m,
                     const double* p0, int32_t n, const double* lb, const double* ub,
                     const jf_opts* opts, jf_result* out);

/* jf_curve_fit_batch — many independent small fits in ONE kernel launch
 * (Gpufit's regime, "slightly faster ... for small data
 * lengths", "runs entirely in CUDA"): fit k minimises
 * 1/2 sum_i (h(y_k,i; x) - z_k,i)^2 by the same TRF as
 * jf_curve_fit, each fit on one warp (pass, subproblem and control), all
 * fits of the batch in one persistent launch.
 *  z: nfits * m doubles, fit k at z + k*m.  y: NULL (implicit grid / t from
 *      opts, the same for every fit), or coordinates per fit (fit k at
 *      y + k*d*m, layout as jf_curve_fit), or — with JF_FLAG_BATCH_SHARED_Y —
 *      one set of d*m coordinates shared by all fits.  opts->sigma (optional):
 *      nfits * m, like z.  Device pointers iff opts->inputs_on_device.
 *  p0: host, nfits * n, or NULL (curve_fit's default p0 for every fit).
 *  lb, ub: n each, shared by all fits, or NULL.
 *  out: host, nfits records, written for every fit: status >= 0 the solver
 *      status, < 0 that fit's error (JF_EINFEASIBLE p0 outside the bounds,
 *      JF_ENONFINITE residuals not finite at p0, JF_EINVAL p0 not finite).
 *  The speculative policy; opts->comm, capacity and trace are not used.
 * Returns 0 (every fit ran; see out[k].status) or a JF_E* error.  Blocks.  */
typedef struct jf_batch_result {
  double x[JF_MAX_N];
  double cost, optimality;
  int32_t status, nfev, njev, nit;
} jf_batch_result;
int32_t jf_curve_fit_batch(int32_t model, const double* y, const double* z, int64_t m, int64_t nfits,
                           const double* p0, int32_t n, const double* lb, const double* ub,
                           const jf_opts* opts, jf_batch_result* out);

/* jf_pass — one J-pass at x (Eq. 1, 2, 4, 5): cost = 1/2 r^T r,
 * grad[n] = J^T r, gram[n*n] = J^T J (row-major, symmetric), *nonfinite =
 * number of points whose residual is not finite.  Any output pointer may be
 * NULL.  x: host, n doubles.  Reads no solver state.  Blocks until done.   */
int32_t jf_pass(int32_t model, const double* y, const double* z, int64_t m,
                const double* x, int32_t n, const jf_opts* opts,
                double* cost, double* grad, double* gram, int32_t* nonfinite);

/* jf_residual_pass — the residual-only pass at x (Eq. 15 numerator):
 * cost = 1/2 r^T r and the non-finite count.  Blocks until done.           */
int32_t jf_residual_pass(int32_t model, const double* y, const double* z, int64_t m,
                         const double* x, int32_t n, const jf_opts* opts,
                         double* cost, int32_t* nonfinite);

/* jf_pass_device — asynchronous J-pass for timing and graph use: all
 * pointers are DEVICE pointers (y may be NULL as above; x_dev: n doubles),
 * the K-vector (layout above) is written to kvec_dev.  residual_only != 0
 * runs the residual-only pass (kvec_dev receives [r^T r, nonfinite]).
 * Enqueued on opts->stream; returns without synchronising.  The launch
 * configuration is the one jf_curve_fit uses.                             */
int32_t jf_pass_device(int32_t model, const double* y, const double* z, int64_t m,
                       const double* x_dev, int32_t n, const jf_opts* opts,
                       int32_t residual_only, double* kvec_dev);

/* jf_trust_region_step — the single-warp subproblem kernel on its own, for
 * parity tests (Alg. 2 + App. B; reading R5-R12).  Given the scaled Gram
 * hatG (n*n, row-major, host), scaled gradient hatg (n), radius Delta and
 * warm-start alpha, m (the number of residuals, for the rank test R6):
 * writes p (n), the final alpha, and the Moré iteration count n_iter
 * (0 = Gauss-Newton step accepted).  Runs on opts->device; blocks.         */
int32_t jf_trust_region_step(const double* hatG, const double* hatg, int32_t n, int64_t m,
                             double Delta, double alpha_in, const jf_opts* opts,
                             double* p, double* alpha_out, int32_t* n_iter);

/* jf_select_step — the device Coleman-Li step selection alone, for parity
 * tests (reading R19/R20; "SciPy's adapted version"): given the scaled
 * quadratic model B_hat (n*n row-major, incl. diag_h on the diagonal) and
 * g_hat, the current x, bounds lb/ub (finite or +-INFINITY), the scaling d and
 * the hat-space trust-region step p_h (n each, host), the radius Delta and
 * theta, writes the chosen step (original space, n), step_h (hat space, n;
 * may be NULL), the predicted reduction -Q(step_h) and the branch (0
 * interior, 1 reflected, 2 truncated, 3 scaled gradient).  Blocks.         */
int32_t jf_select_step(const double* hatB, const double* hatg, const double* x, const double* lb,
                       const double* ub, const double* d, const double* p_h, int32_t n, double Delta,
                       double theta, const jf_opts* opts, double* step, double* step_h, double* pred,
                       int32_t* branch);

/* Multi-GPU: data-parallel sharding over m (one process per GPU).  Each rank
 * owns a mailbox in its device memory; jf_comm_export() writes an IPC handle
 * for it, the caller all-gathers the handles (e.g. with torch.distributed),
 * and jf_comm_connect() maps every peer's mailbox.  Inside each pass kernel
 * the last block pushes its K-vector into every peer's mailbox over NVLink
 * and sums the R vectors in rank order (deterministic, identical on all
 * ranks), so the n x n subproblem runs redundantly and identically on every
 * rank with no host round trip.  jf_comm_create_local() instead makes R
 * virtual ranks on ONE device (sequential-free emulation for tests).       */
int32_t jf_comm_create(int32_t rank, int32_t nranks, int32_t device, jf_comm** comm);
int32_t jf_comm_export(const jf_comm* comm, uint8_t handle[JF_COMM_HANDLE_BYTES]);
int32_t jf_comm_connect(jf_comm* comm, const uint8_t* all_handles /* nranks * JF_COMM_HANDLE_BYTES */);
int32_t jf_comm_create_local(int32_t nranks, int32_t device, jf_comm** comms /* nranks out */);
int32_t jf_comm_destroy(jf_comm* comm);
/* A pass kernel whose peers do not all arrive within timeout_ms reports
 * JF_ECOMM (jf_pass*) or ends the fit with status JF_ECOMM instead of
 * waiting forever.  Default 20000 ms.  Returns 0 or JF_EINVAL.              */
int32_t jf_comm_set_timeout(jf_comm* comm, int32_t timeout_ms);
/* One cross-rank combine of a KMAX-double vector through the mailboxes (the
 * exchange every pass kernel ends with), timed on the device: *us receives
 * the mean microseconds per combine over `reps` back-to-back combines of
 * value v; *sum receives the rank-ordered sum of v over the ranks.  All
 * ranks must call it together.  For latency measurements.  */
int32_t jf_comm_bench(jf_comm* comm, double v, int32_t reps, double* sum, double* us);

/* Drop every instantiated fit graph of `device` (the next fit builds afresh). */
int32_t jf_graph_cache_clear(int32_t device);

/* Human-readable name of a return code (static storage). */
const char* jf_strerror(int32_t code);

/* Library build identifier (static storage), e.g. "jfb200 sm_100a". */
const char* jf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* JF_H_ */

// jf_host.cu — host driver and C ABI of libjfb200.so (include/jf.h).
//
// Responsibilities: validate input (reading R18), stage
// host data into HBM, pick the kernel instance for (model, coordinate mode),
// size the grid, and run a fit either as ONE CUDA-graph launch — a WHILE
// conditional node whose body is the pass kernel(s); the last block of each
// pass runs the solver step and sets the loop condition on the device — or as
// a host-driven loop (use_graph = 0).  Graphs are cached per (model, mode,
// grid, policy) and replayed for any data, so only the first fit pays the
// instantiation (cf. JAX tracing).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/jf.h"
#include "jf_kernels.h"
#include "jf_state.cuh"

#ifndef JF_DEV
#define JF_DEV 0
#endif

using namespace jf;

namespace {
// NVTX ranges (SURVEY §5 tracing): per fit, per pass call, and in the host-
// driven loop per pass / solver launch; visible in Nsight Systems, free when
// no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

namespace jf {  // jf_comm.cu
int launch_comm_sum(const CommDev& cd, unsigned long long epoch, double v, double* d_out, int* d_err, cudaStream_t s);
const void* comm_sum_kernel_ptr();
}  // namespace jf

namespace jf {  // jf_solver.cu
const void* solver_kernel_ptr();
int launch_solver(FitState* st, const double* kv, cudaStream_t s);
int launch_tr_step(const double* hatG, const double* hatg, int n, int64_t m, double Delta, double alpha_in,
                   double* out, int dbg, cudaStream_t s);
int launch_select_step(const double* in, int n, double Delta, double theta, double* out, cudaStream_t s);
}  // namespace jf

// A rank's view of the multi-GPU mailboxes (jf.h jf_comm_*).
struct jf_comm {
  int rank = 0, nranks = 1, device = 0;
  unsigned long long epoch = 0;
  void* mbox = nullptr;           // local mailbox (device)
  bool owns_mbox = true;
  bool local = false;             // created by jf_comm_create_local
  void* peer[8] = {nullptr};      // mapped mailboxes of all ranks
  bool opened[8] = {false};
  unsigned long long timeout_ns = 20000000000ull;  // jf_comm_set_timeout
};

namespace {

Kernels get_kernels(int model, int coord) {
  switch (model) {
    case JF_LINEAR: return kernels_linear(coord);
    case JF_EXP_DECAY: return kernels_exp_decay(coord);
    case JF_GAUSS1D: return kernels_gauss1d(coord);
    case JF_GAUSS2D_ROT: return kernels_gauss2d(coord);
    case JF_GAUSS2D_ROT_X2: return kernels_gauss2d_x2(coord);
    default: return Kernels{};
  }
}

__global__ void inv_kernel(double* p, int64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 1.0 / p[i];
}

// Wait for the stream by polling (a blocking cudaStreamSynchronize may sleep
// and wake up tens of microseconds late: a fit is ~0.1-0.4 ms).
cudaError_t stream_wait(cudaStream_t s) {
  for (;;) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e != cudaErrorNotReady) return e;
  }
}

int model_n(int model) {
  switch (model) {
    case JF_LINEAR: return 2;
    case JF_EXP_DECAY: return 3;
    case JF_GAUSS1D: return 4;
    case JF_GAUSS2D_ROT: return 7;
    case JF_GAUSS2D_ROT_X2: return 13;
    default: return -1;
  }
}
int model_d(int model) {
  switch (model) {
    case JF_LINEAR:
    case JF_EXP_DECAY:
    case JF_GAUSS1D: return 1;
    case JF_GAUSS2D_ROT:
    case JF_GAUSS2D_ROT_X2: return 2;
    default: return -1;
  }
}

#define CK(call)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) {                                                                     \
      fprintf(stderr, "jfb200: %s failed: %s (%s:%d)\n", #call, cudaGetErrorString(e_), __FILE__, \
              __LINE__);                                                                         \
      return e_ == cudaErrorMemoryAllocation ? JF_ENOMEM : JF_ECUDA;                             \
    }                                                                                            \
  } while (0)

struct GraphKey {
  const void* jk;
  int policy, jgrid, rgrid, qr;
  bool operator<(const GraphKey& o) const {
    return std::tie(jk, policy, jgrid, rgrid, qr) < std::tie(o.jk, o.policy, o.jgrid, o.rgrid, o.qr);
  }
};

struct Ctx {
  std::mutex mu;
  bool ready = false;
  int dev = 0;
  int nsm = 148;
  cudaStream_t stream = nullptr;
  PassArgs* d_args = nullptr;
  PassArgs* h_args = nullptr;  // pinned: last upload to d_args (a repeated fit skips the copy)
  // Pinned staging for every small host<->device copy: a pageable copy is
  // synchronous inside the driver and can stall other threads' launches while
  // it waits — fatal when those threads' ranks spin on a combine with ours.
  double* h_pin = nullptr;
  bool h_args_valid = false;
  FitState* d_state = nullptr;
  FitState* h_state = nullptr;  // pinned
  double* d_partials = nullptr;
  int partial_blocks = 0;
  unsigned int* d_ticket = nullptr;
  double* d_out = nullptr;  // KMAX
  double* d_x = nullptr;    // NMAX
  double* d_trace = nullptr;
  int trace_cap = 0;
  double* d_in = nullptr;  // staged host inputs
  size_t in_cap = 0;
  double* d_scratch = nullptr;  // small per-call scratch (status word, subproblem I/O)
  QRState* d_qr = nullptr;      // TSQR working set
  std::map<GraphKey, cudaGraphExec_t> graphs;
  // Calls may run on different streams but share the buffers above: each
  // call waits for the previous call's work (event on its stream) before it
  // enqueues anything, and records its own completion.
  cudaEvent_t done = nullptr;
  cudaStream_t done_stream = nullptr;
  // batched fits (jf_curve_fit_batch)
  FitState* d_tmpl = nullptr;
  QRState* d_qr_batch = nullptr;
  int qr_batch_cap = 0;
  BatchResult* d_bout = nullptr;
  size_t bout_cap = 0;
};

// Contexts: [0, 64) one per device; [64, 64 + 64*8) per (device, virtual rank)
// of a jf_comm_create_local emulation, so emulated ranks run concurrently.
Ctx g_ctx[64 + 64 * 8];
constexpr int SCRATCH_DOUBLES = 1024;
constexpr int PIN_DOUBLES = 1024;
constexpr int TICKETS = 128;  // grid_reduce: [0] groups, [1 + g] blocks of group g (<= 127 groups)

void preload_kernels();

int ctx_init(Ctx& c, int dev) {
  if (c.ready) return 0;
  CK(cudaSetDevice(dev));
  c.dev = dev;
  CK(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  {
    static std::mutex attr_mu;
    static bool attr_done[64] = {};
    std::lock_guard<std::mutex> g(attr_mu);
    if (!attr_done[dev]) {
      kernel_attrs_init();
      kernel_attrs_init_x2();
      preload_kernels();
      attr_done[dev] = true;
    }
  }
  CK(cudaMalloc(&c.d_args, sizeof(PassArgs)));
  CK(cudaMalloc(&c.d_state, sizeof(FitState)));
  CK(cudaMallocHost(&c.h_state, sizeof(FitState)));
  CK(cudaMallocHost(&c.h_args, sizeof(PassArgs)));
  CK(cudaMallocHost(&c.h_pin, sizeof(double) * PIN_DOUBLES));
  c.partial_blocks = c.nsm * 4;
  // block rows + group rows of the two-level grid reduction (jf_pass.cuh grid_reduce)
  CK(cudaMalloc(&c.d_partials, sizeof(double) * (size_t)(c.partial_blocks + c.partial_blocks / 16 + 1) * KMAX));
  CK(cudaMalloc(&c.d_ticket, sizeof(unsigned int) * TICKETS));
  CK(cudaMalloc(&c.d_out, sizeof(double) * KMAX));
  CK(cudaMalloc(&c.d_x, sizeof(double) * NMAX));
  CK(cudaMalloc(&c.d_scratch, sizeof(double) * SCRATCH_DOUBLES));
  CK(cudaMalloc(&c.d_qr, sizeof(QRState)));
  CK(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
  // no device-wide synchronisation here: emulated ranks (jf_comm_create_local)
  // may have pass kernels spinning on their mailboxes while a peer initialises
  CK(cudaMemsetAsync(c.d_ticket, 0, sizeof(unsigned int) * TICKETS, c.stream));
  CK(cudaMemsetAsync(c.d_scratch, 0, sizeof(double) * SCRATCH_DOUBLES, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  c.ready = true;
  return 0;
}

// Load every kernel a fit or pass can launch into the context now (CUDA
// loads modules lazily at a function's first launch, and loading waits for
// running kernels: a rank whose first launch of a kernel happens while a peer
// rank's kernel spins on its mailbox would stall until that peer times out).
void preload_kernels() {
  cudaFuncAttributes fa;
  auto touch = [&](const void* f) {
    if (f) cudaFuncGetAttributes(&fa, f);
  };
  for (int model = 0; model <= JF_GAUSS2D_ROT_X2; ++model)
    for (int coord = 0; coord <= COORD_IMPLICIT_T; ++coord) {
      const Kernels k = get_kernels(model, coord);
      for (KernelFn f : {k.jk, k.rk, k.jkw, k.rkw}) touch((const void*)f);
      touch((const void*)k.small);
      touch((const void*)k.smallw);
    }
  touch(solver_kernel_ptr());
  touch(comm_sum_kernel_ptr());
  touch((const void*)inv_kernel);
  cudaGetLastError();
}

// The grid of a pass kernel: enough blocks to fill every SM at the kernel's
// occupancy, fewer for small m.  A pure function of (kernel, m): fixed
// reduction order, bitwise reproducible passes (H4).
std::mutex g_occ_mu;
std::map<std::pair<int, const void*>, int> g_occ;  // (device, kernel) -> resident blocks/SM

int grid_for(Ctx& c, KernelFn f, int tpb, int64_t m, int smem = 0) {
  int occ;
  {
    std::lock_guard<std::mutex> g(g_occ_mu);
    auto key = std::make_pair(c.dev, (const void*)f);
    auto it = g_occ.find(key);
    if (it == g_occ.end()) {
      occ = 1;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, tpb, smem) != cudaSuccess || occ < 1) occ = 1;
      if (occ > 4) occ = 4;
      g_occ[key] = occ;
    } else {
      occ = it->second;
    }
  }
  const int64_t need = (m + tpb - 1) / tpb;
  int64_t g = (int64_t)c.nsm * occ;
  if (need < g) g = need;
  if (g < 1) g = 1;
  return (int)g;
}

// The point count launch shapes are sized for: the capacity when one is set
// (jf_opts.capacity, N3: one cached graph serves every m <= capacity).
int64_t pass_grid_m(const jf_opts& o, int64_t m) { return o.capacity > 0 ? o.capacity : m; }

const PassArgs g_zero_args = {};  // the by-value args of launches that read device-resident ones

// The two pass kernels a call uses, with their launch shapes.
struct PassPair {
  KernelFn j = nullptr, r = nullptr;
  int jtpb = 256, rtpb = 256, jgrid = 1, rgrid = 1, jsmem = 0;
  bool fused = false;  // j runs the solver step in its last block (speculative fits)
};

PassPair select_pass(Ctx& c, const Kernels& k, bool weighted, int64_t m) {
  PassPair p;
  p.j = weighted ? k.jkw : k.jk;
  p.r = weighted ? k.rkw : k.rk;
  p.jtpb = (weighted && k.jwtpb > 0) ? k.jwtpb : k.jtpb;
  p.rtpb = k.rtpb;
  p.jsmem = weighted ? 0 : k.jsmem;
  p.fused = !weighted && k.jfused;
  p.jgrid = grid_for(c, p.j, p.jtpb, m, p.jsmem);
  const bool jsplit = (weighted && k.jwsplit >= 0) ? (k.jwsplit != 0) : k.jsplit;
  if (jsplit) {  // two equal halves
    p.jgrid = p.jgrid < 2 ? 2 : p.jgrid + (p.jgrid & 1);
  }
  p.rgrid = grid_for(c, p.r, p.rtpb, m);
  return p;
}

}  // namespace

namespace {

constexpr size_t MBOX_DATA_BYTES(int R) { return sizeof(double) * 2 * (size_t)R * KMAX; }
size_t mbox_bytes(int R) { return MBOX_DATA_BYTES(R) + sizeof(unsigned long long) * 8; }

void fill_comm(CommDev& cd, const jf_comm* cm) {
  memset(&cd, 0, sizeof(cd));
  cd.rank = cm->rank;
  cd.nranks = cm->nranks;
  for (int p = 0; p < cm->nranks; ++p) {
    char* base = (char*)cm->peer[p];
    cd.mbox_data[p] = (double*)base;
    cd.mbox_flag[p] = (unsigned long long*)(base + MBOX_DATA_BYTES(cm->nranks));
  }
  cd.epoch = cm->epoch;
  cd.timeout_ns = cm->timeout_ns;
}

struct Staged {
  const double* z = nullptr;
  const double* y0 = nullptr;
  const double* y1 = nullptr;
  const double* wsig = nullptr;
  int coord = COORD_EXPLICIT;
  double upload_s = 0.0;
};

// Grow a device buffer with the stream-ordered allocator (no device-wide
// synchronisation, which could stall against emulated ranks' kernels).
int ensure(double*& p, size_t& cap, size_t need, cudaStream_t s) {
  if (cap >= need) return 0;
  if (p) CK(cudaFreeAsync(p, s));
  p = nullptr;
  cap = 0;
  CK(cudaMallocAsync((void**)&p, sizeof(double) * need, s));
  cap = need;
  return 0;
}


// Validate the data description and make y/z/sigma available in HBM.
int stage_inputs(Ctx& c, cudaStream_t s, int model, const double* y, const double* z, int64_t m,
                 const jf_opts& o, Staged& st) {
  const int d = model_d(model);
  if (d < 0 || z == nullptr || m < 1) return JF_EINVAL;
  int coord;
  if (y != nullptr) {
    coord = COORD_EXPLICIT;
  } else if (d == 2) {
    if (o.grid_w < 1 || o.grid_h < 1 || o.grid_w * o.grid_h != m) return JF_EINVAL;
    coord = COORD_GRID;
  } else {
    if (!(o.dt == o.dt) || !std::isfinite(o.t0) || !std::isfinite(o.dt)) return JF_EINVAL;
    coord = COORD_IMPLICIT_T;
  }
  st.coord = coord;
  const size_t ny = (coord == COORD_EXPLICIT) ? (size_t)d * m : 0;
  const size_t nw = o.sigma ? (size_t)m : 0;
  auto t0 = std::chrono::steady_clock::now();
  if (o.inputs_on_device) {
    st.z = z;
    if (coord == COORD_EXPLICIT) {
      st.y0 = y;
      st.y1 = (d == 2) ? y + m : nullptr;
    }
    if (o.sigma) {  // 1/sigma needs a scratch copy
      if (int e = ensure(c.d_in, c.in_cap, nw, s)) return e;
      CK(cudaMemcpyAsync(c.d_in, o.sigma, sizeof(double) * nw, cudaMemcpyDeviceToDevice, s));
      inv_kernel<<<c.nsm * 4, 256, 0, s>>>(c.d_in, m);
      CK(cudaGetLastError());
      st.wsig = c.d_in;
    }
  } else {
    const size_t need = (size_t)m + ny + nw;
    if (int e = ensure(c.d_in, c.in_cap, need, s)) return e;
    double* p = c.d_in;
    CK(cudaMemcpyAsync(p, z, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    st.z = p;
    p += m;
    if (ny) {
      CK(cudaMemcpyAsync(p, y, sizeof(double) * ny, cudaMemcpyHostToDevice, s));
      st.y0 = p;
      st.y1 = (d == 2) ? p + m : nullptr;
      p += ny;
    }
    if (nw) {
      CK(cudaMemcpyAsync(p, o.sigma, sizeof(double) * nw, cudaMemcpyHostToDevice, s));
      inv_kernel<<<c.nsm * 4, 256, 0, s>>>(p, m);
      CK(cudaGetLastError());
      st.wsig = p;
    }
    CK(cudaStreamSynchronize(s));
  }
  st.upload_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return 0;
}

void fill_args(PassArgs& a, const Staged& sg, int64_t m, const jf_opts& o) {
  memset(&a, 0, sizeof(a));  // padding too: fit args are compared bytewise with the last upload
  a.z = sg.z;
  a.y0 = sg.y0;
  a.y1 = sg.y1;
  a.wsig = sg.wsig;
  a.m = m;
  a.W = o.grid_w;
  a.row0 = o.grid_row0;
  a.index0 = o.index0;
  a.t0 = o.t0;
  a.dt = o.dt;
  a.coord = sg.coord;
}

struct Lock {
  Ctx* c = nullptr;
  std::unique_lock<std::mutex> lk;
};

int acquire(const jf_opts& o, Ctx*& c, std::unique_lock<std::mutex>& lk, cudaStream_t& s) {
  if (o.device < 0 || o.device >= 64) return JF_EINVAL;
  if (o.comm && o.comm->local) c = &g_ctx[64 + o.device * 8 + o.comm->rank];
  else c = &g_ctx[o.device];
  lk = std::unique_lock<std::mutex>(c->mu);
  if (cudaSetDevice(o.device) != cudaSuccess) return JF_ECUDA;
  int r = ctx_init(*c, o.device);
  if (r) return r;
  s = o.stream ? (cudaStream_t)o.stream : c->stream;
  return 0;
}

// host-side strict feasibility, rstep = 1e-10 (reading R18/R19: x0 of the bounded path)
void strictly_feasible_host(double* x, const double* lb, const double* ub, int n, double rstep) {
  for (int j = 0; j < n; ++j) {
    const double lo = lb[j], hi = ub[j], v = x[j];
    double xn = v;
    if (rstep == 0.0) {
      if (v <= lo) xn = nextafter(lo, hi);
      else if (v >= hi) xn = nextafter(hi, lo);
    } else {
      const double ld = v - lo, ud = hi - v;
      const double lt = rstep * fmax(1.0, fabs(lo)), ut = rstep * fmax(1.0, fabs(hi));
      if (std::isfinite(lo) && ld <= fmin(ud, lt)) xn = lo + lt;
      else if (std::isfinite(hi) && ud <= fmin(ld, ut)) xn = hi - ut;
    }
    if (xn < lo || xn > hi) xn = 0.5 * (lo + hi);
    x[j] = xn;
  }
}

void active_mask_host(const double* x, const double* lb, const double* ub, int n, double rtol, int8_t* act) {
  for (int j = 0; j < n; ++j) {
    act[j] = 0;
    const double ld = x[j] - lb[j], ud = ub[j] - x[j];
    const double lt = rtol * fmax(1.0, fabs(lb[j])), ut = rtol * fmax(1.0, fabs(ub[j]));
    if (std::isfinite(lb[j]) && ld <= fmin(ud, lt)) act[j] = -1;
    if (std::isfinite(ub[j]) && ud <= fmin(ld, ut)) act[j] = 1;
  }
}

// One pass kernel launch: d_args (device-resident, fits) or, with d_args ==
// nullptr, the arguments by value (plain passes: immutable once enqueued or
// captured into a graph).
int launch_pass(const PassPair& k, bool jac, cudaStream_t s, const PassArgs* d_args, FitState* d_state,
                const PassArgs& av) {
  KernelFn f = jac ? k.j : k.r;
  const int grid = jac ? k.jgrid : k.rgrid;
  const int tpb = jac ? k.jtpb : k.rtpb;
  const int smem = jac ? k.jsmem : 0;
  f<<<grid, tpb, smem, s>>>(d_args, d_state, (cudaGraphConditionalHandle)0, 0, av);
  CK(cudaGetLastError());
  return 0;
}

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// Stream ordering of the context's shared buffers across calls (see Ctx::done).
struct StreamOrder {
  Ctx* c = nullptr;
  cudaStream_t s = nullptr;
  bool cap = false;
  int begin(Ctx* c_, cudaStream_t s_) {
    c = c_;
    s = s_;
    cap = capturing(s);
    if (!cap && c->done_stream && c->done_stream != s) CK(cudaStreamWaitEvent(s, c->done, 0));
    return 0;
  }
  ~StreamOrder() {
    if (c && !cap && cudaEventRecord(c->done, s) == cudaSuccess) c->done_stream = s;
  }
};

int build_graph(Ctx& c, const PassPair& k, int policy, bool qr, bool fused, cudaGraphExec_t* out) {
  (void)qr;
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  // the fit's initial state in (the host-written prefix) and the final state
  // out are nodes of the graph too: one launch per fit
  cudaGraphNode_t up, cn, down;
  CK(cudaGraphAddMemcpyNode1D(&up, g, nullptr, 0, c.d_state, c.h_state, FITSTATE_UPLOAD, cudaMemcpyHostToDevice));
  CK(cudaGraphAddNode(&cn, g, &up, 1, &cp));
  CK(cudaGraphAddMemcpyNode1D(&down, g, &cn, 1, c.h_state, c.d_state, sizeof(FitState), cudaMemcpyDeviceToHost));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  int use = 1;
  PassArgs* pa = c.d_args;
  FitState* st = c.d_state;
  const double* kv = c.d_out;
  PassArgs av;
  memset(&av, 0, sizeof(av));  // unused: the fit's args are read from pa
  void* pargs[5] = {&pa, &st, &h, &use, &av};
  void* sargs[4] = {&st, &kv, &h, &use};
  cudaKernelNodeParams kp;
  memset(&kp, 0, sizeof(kp));
  cudaKernelNodeParams sp;
  memset(&sp, 0, sizeof(sp));
  sp.func = const_cast<void*>(solver_kernel_ptr());
  sp.gridDim = dim3(1);
  sp.blockDim = dim3(32);
  sp.kernelParams = sargs;
  // body: [r-pass -> solver ->] J-pass -> solver; each pass kernel runs only
  // when the state's phase asks for it, each solver only after a pass ran
  // solver nodes depend programmatically on the pass before them (PDL): the
  // solver kernel is scheduled while the pass drains and waits in
  // griddepcontrol.wait for its results, hiding the launch latency
  // Every kernel after the first depends programmatically on the one before
  // (PDL): it is scheduled while its predecessor runs and waits in
  // griddepcontrol.wait for the predecessor's completion and memory.
  cudaGraphNode_t prev = nullptr;
  bool prev_is_pass = false;
  auto add = [&](const cudaKernelNodeParams& p, bool is_solver) -> int {
    cudaGraphNode_t nd;
    (void)prev_is_pass;
    if (prev) {
      cudaGraphNodeParams np = {};
      np.type = cudaGraphNodeTypeKernel;
      np.kernel.func = p.func;
      np.kernel.gridDim = p.gridDim;
      np.kernel.blockDim = p.blockDim;
      np.kernel.sharedMemBytes = p.sharedMemBytes;
      np.kernel.kernelParams = p.kernelParams;
      cudaGraphEdgeData ed = {};
      ed.from_port = cudaGraphKernelNodePortProgrammatic;
      ed.to_port = cudaGraphKernelNodePortDefault;
      ed.type = cudaGraphDependencyTypeProgrammatic;
      CK(cudaGraphAddNode_v2(&nd, body, &prev, &ed, 1, &np));
    } else {
      CK(cudaGraphAddKernelNode(&nd, body, prev ? &prev : nullptr, prev ? 1 : 0, &p));
    }
    prev = nd;
    prev_is_pass = !is_solver;
    return 0;
  };
  kp.kernelParams = pargs;
  // U copies of the iteration per trip of the WHILE loop: the conditional
  // node's per-trip overhead (~6 us) is paid once per U iterations; copies
  // after the fit ended find nothing to do (phase DONE) and return at once
  // (~3 us for a fused J-pass: it drains its first bulk copies).  Fused
  // bodies (one kernel per trial): 6, so a 6-pass fit (T, C3) is one trip.
  const int unroll = fused ? 6 : 3;
  for (int u = 0; u < unroll; ++u) {
    if (policy == JF_POLICY_CONSERVATIVE) {
      kp.func = (void*)k.r;
      kp.gridDim = dim3(k.rgrid);
      kp.blockDim = dim3(k.rtpb);
      if (int e = add(kp, false)) return e;
      if (int e = add(sp, true)) return e;
    }
    // (TSQR: the J-pass kernel also runs the preconditioned second pass when
    // the phase is PH_QR2 — no separate node)
    kp.func = (void*)k.j;
    kp.gridDim = dim3(k.jgrid);
    kp.blockDim = dim3(k.jtpb);
    kp.sharedMemBytes = k.jsmem;
    if (int e = add(kp, false)) return e;
    kp.sharedMemBytes = 0;
    if (!fused)  // (fused: the J-pass's last block runs the solver step)
      if (int e = add(sp, true)) return e;
  }
  CK(cudaGraphInstantiate(out, g, 0));
  cudaGraphDestroy(g);
  return 0;
}

}  // namespace

// =============================================================== C ABI
extern "C" {

void jf_opts_default(jf_opts* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->ftol = o->xtol = o->gtol = 1e-8;
  o->max_nfev = 0;
  o->x_scale_mode = JF_XSCALE_JAC;
  o->solver = JF_SOLVE_AUTO;
  o->policy = JF_POLICY_SPECULATIVE;
  o->t0 = 0.0;
  o->dt = 1.0;
  o->use_graph = 1;
}

int32_t jf_model_nparams(int32_t model) { return model_n(model); }
int32_t jf_model_ydim(int32_t model) { return model_d(model); }
int32_t jf_model_kslots(int32_t model) {
  const int n = model_n(model);
  return n < 0 ? -1 : tri_count(n) + 1;
}

const char* jf_strerror(int32_t code) {
  switch (code) {
    case 0: return "max_nfev reached";
    case 1: return "gtol satisfied";
    case 2: return "ftol satisfied";
    case 3: return "xtol satisfied";
    case 4: return "ftol and xtol satisfied";
    case JF_EINVAL: return "invalid argument";
    case JF_EINFEASIBLE: return "initial guess outside the bounds";
    case JF_ENONFINITE: return "residuals not finite at the initial guess";
    case JF_ECUDA: return "CUDA error";
    case JF_ECOMM: return "multi-GPU combine failed";
    case JF_ENOMEM: return "out of memory";
    default: return "unknown code";
  }
}

const char* jf_version(void) { return "jfb200 0.1 sm_100a"; }

static int pass_common(int32_t model, const double* y, const double* z, int64_t m, const double* x, int x_on_device,
                       int32_t n, const jf_opts* opts, int residual_only, double* out_dev_or_null,
                       double* host_out /* KMAX */, bool sync) {
  NvtxRange nv(residual_only ? "jf_residual_pass" : "jf_pass");
  jf_opts o;
  if (opts) o = *opts;
  else jf_opts_default(&o);
  if (model_n(model) < 0 || n != model_n(model) || !x || !z || m < 1) return JF_EINVAL;
  Ctx* c;
  std::unique_lock<std::mutex> lk;
  cudaStream_t s;
  int r = acquire(o, c, lk, s);
  if (r) return r;
  StreamOrder order;
  if ((r = order.begin(c, s))) return r;
  Staged sg;
  r = stage_inputs(*c, s, model, y, z, m, o, sg);
  if (r) return r;
  Kernels kk = get_kernels(model, sg.coord);
  if (!kk.jk) return JF_EINVAL;
  const PassPair k = select_pass(*c, kk, sg.wsig != nullptr, pass_grid_m(o, m));
  PassArgs a;
  fill_args(a, sg, m, o);
  a.epilogue = EPI_NONE;
  a.no_chain = (o.flags & JF_FLAG_ALT_COORDS) ? 1 : 0;
#if JF_DEV  // development builds: per-warp timeline of the moment J-pass (tools/stamps2.py)
  const char* stamps = (residual_only || order.cap) ? nullptr : getenv("JF_DEBUG_STAMPS");
  static unsigned long long* d_dbg = nullptr;
  constexpr int DBG_N = 4 * 16384;
  if (stamps && !d_dbg) CK(cudaMalloc(&d_dbg, sizeof(unsigned long long) * DBG_N));
  a.dbg = stamps ? d_dbg : nullptr;
  if (stamps) CK(cudaMemsetAsync(d_dbg, 0, sizeof(unsigned long long) * DBG_N, s));
#endif
  if (x_on_device) {
    a.x = x;
    if (o.x_host && model == JF_GAUSS2D_ROT) {  // (the caller's host copy of x_dev)
      gauss2d_prologue(o.x_host, a.pre);
      a.has_pre = 1;
    } else if (o.x_host && model == JF_GAUSS2D_ROT_X2) {
      gauss2d_x2_prologue(o.x_host, a.pre);
      a.has_pre = 1;
    }
  } else {
    if (model == JF_GAUSS2D_ROT) {  // the moment J-pass's prologue, once, here
      gauss2d_prologue(x, a.pre);
      a.has_pre = 1;
    } else if (model == JF_GAUSS2D_ROT_X2) {
      gauss2d_x2_prologue(x, a.pre);
      a.has_pre = 1;
    }
    double* hx = c->h_pin + 512;  // (the previous call's copy finished: calls are stream-ordered)
    memcpy(hx, x, sizeof(double) * n);
    CK(cudaMemcpyAsync(c->d_x, hx, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    a.x = c->d_x;
  }
  a.partials = c->d_partials;
  a.ticket = c->d_ticket;
  a.out = out_dev_or_null ? out_dev_or_null : c->d_out;
  a.err = (int*)c->d_scratch;
  if (o.comm) {
    a.use_comm = 1;
    fill_comm(a.comm, o.comm);
    o.comm->epoch += 1;
  }
  // the arguments travel by value with the launch (immutable once enqueued
  // or captured into a graph)
  r = launch_pass(k, !residual_only, s, nullptr, c->d_state, a);
  if (r) return r;
#if JF_DEV
  if (stamps) {
    static unsigned long long h_dbg[DBG_N];
    CK(cudaMemcpyAsync(h_dbg, d_dbg, sizeof(h_dbg), cudaMemcpyDeviceToHost, s));
    CK(stream_wait(s));
    if (FILE* f = fopen(stamps, "wb")) {
      fwrite(h_dbg, sizeof(h_dbg), 1, f);
      fclose(f);
    }
  }
#endif
  const int KSo = residual_only ? 2 : tri_count(n) + 1;
  if (host_out) CK(cudaMemcpyAsync(c->h_pin, a.out, sizeof(double) * KSo, cudaMemcpyDeviceToHost, s));
  if (sync) {
    int* herr = (int*)(c->h_pin + 256);
    CK(cudaMemcpyAsync(herr, a.err, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(stream_wait(s));
    const int err = *herr;
    if (host_out) memcpy(host_out, c->h_pin, sizeof(double) * KSo);
    if (err) {
      CK(cudaMemsetAsync(a.err, 0, sizeof(int), s));
      CK(stream_wait(s));
      return err;
    }
  }
  return 0;
}

int32_t jf_pass(int32_t model, const double* y, const double* z, int64_t m, const double* x, int32_t n,
                const jf_opts* opts, double* cost, double* grad, double* gram, int32_t* nonfinite) {
  double kv[KMAX];
  int r = pass_common(model, y, z, m, x, 0, n, opts, 0, nullptr, kv, true);
  if (r) return r;
  if (cost) *cost = 0.5 * kv[tri_slot(n, n, n)];
  for (int j = 0; j < n; ++j) {
    if (grad) grad[j] = kv[tri_slot(n, j, n)];
    for (int k = 0; k < n; ++k)
      if (gram) gram[j * n + k] = kv[tri_slot(n, j < k ? j : k, j < k ? k : j)];
  }
  if (nonfinite) *nonfinite = (int32_t)kv[tri_count(n)];
  return 0;
}

int32_t jf_residual_pass(int32_t model, const double* y, const double* z, int64_t m, const double* x, int32_t n,
                         const jf_opts* opts, double* cost, int32_t* nonfinite) {
  double kv[KMAX];
  int r = pass_common(model, y, z, m, x, 0, n, opts, 1, nullptr, kv, true);
  if (r) return r;
  if (cost) *cost = 0.5 * kv[0];
  if (nonfinite) *nonfinite = (int32_t)kv[1];
  return 0;
}

int32_t jf_pass_device(int32_t model, const double* y, const double* z, int64_t m, const double* x_dev, int32_t n,
                       const jf_opts* opts, int32_t residual_only, double* kvec_dev) {
  jf_opts o;
  if (opts) o = *opts;
  else jf_opts_default(&o);
  if (!o.inputs_on_device || !kvec_dev) return JF_EINVAL;
  return pass_common(model, y, z, m, x_dev, 1, n, &o, residual_only, kvec_dev, nullptr, false);
}

static int32_t fit_impl(int32_t model, const double* y, const double* z, int64_t m, const double* p0, int32_t n,
                        const double* lb, const double* ub, const jf_opts* opts, jf_result* out) {
  NvtxRange nv("jf_curve_fit");
#if JF_DEV  // development: host-side phase times of a fit (stderr)
  const auto hd0 = std::chrono::steady_clock::now();
  auto hdt = [&]() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - hd0).count(); };
  double hd[8] = {0};
#define JF_HSTAMP(i) hd[i] = hdt()
#else
#define JF_HSTAMP(i) (void)0
#endif
  auto fail = [&](int code) {
    out->status = code;
    return code;
  };
  jf_opts o;
  if (opts) o = *opts;
  else jf_opts_default(&o);
  if (model_n(model) < 0 || n != model_n(model) || !z || m < 1) return fail(JF_EINVAL);
  if (o.comm && o.m_global != 0 && o.m_global < m) return fail(JF_EINVAL);
  if (o.capacity < 0 || (o.capacity > 0 && o.capacity < m)) return fail(JF_EINVAL);
  out->n = n;
  // ---- bounds and initial point (R18, R19)
  double L[NMAX], U[NMAX], X0[NMAX], XS[NMAX];
  bool bounded = false;
  for (int j = 0; j < n; ++j) {
    L[j] = lb ? lb[j] : -INFINITY;
    U[j] = ub ? ub[j] : INFINITY;
    if (std::isnan(L[j]) || std::isnan(U[j]) || !(L[j] < U[j])) return fail(JF_EINVAL);
    if (std::isfinite(L[j]) || std::isfinite(U[j])) bounded = true;
  }
  for (int j = 0; j < n; ++j) {
    if (p0) {
      X0[j] = p0[j];
    } else {  // curve_fit's default initial guess
      const bool lf = std::isfinite(L[j]), uf = std::isfinite(U[j]);
      X0[j] = (lf && uf) ? 0.5 * (L[j] + U[j]) : (lf ? L[j] + 1.0 : (uf ? U[j] - 1.0 : 1.0));
    }
    if (!std::isfinite(X0[j])) return fail(JF_EINVAL);
    if (X0[j] < L[j] || X0[j] > U[j]) return fail(JF_EINFEASIBLE);
  }
  if (o.x_scale_mode == JF_XSCALE_ARRAY) {
    if (!o.x_scale) return fail(JF_EINVAL);
    for (int j = 0; j < n; ++j) {
      if (!std::isfinite(o.x_scale[j]) || !(o.x_scale[j] > 0)) return fail(JF_EINVAL);
      XS[j] = 1.0 / o.x_scale[j];
    }
  } else {
    for (int j = 0; j < n; ++j) XS[j] = 1.0;
  }
  if (o.x_scale_mode < 0 || o.x_scale_mode > 2 || o.policy < 0 || o.policy > 1 || o.solver < 0 || o.solver > 2)
    return fail(JF_EINVAL);
  if (bounded) strictly_feasible_host(X0, L, U, n, 1e-10);

  Ctx* c;
  std::unique_lock<std::mutex> lk;
  cudaStream_t s;
  int r = acquire(o, c, lk, s);
  if (r) return fail(r);
  StreamOrder order;
  if ((r = order.begin(c, s))) return fail(r);
  if (order.cap) return fail(JF_EINVAL);  // a fit synchronises: it cannot be captured
  Staged sg;
  {
    NvtxRange nv2("stage_inputs");
    r = stage_inputs(*c, s, model, y, z, m, o, sg);
  }
  if (r) return fail(r);
  out->t_upload_s = sg.upload_s;
  Kernels kk = get_kernels(model, sg.coord);
  if (!kk.jk) return fail(JF_EINVAL);
  const int64_t mg = pass_grid_m(o, m);  // launch shapes are sized for the capacity (N3)
  const PassPair k = select_pass(*c, kk, sg.wsig != nullptr, mg);
  int64_t m_global = m;
  if (o.comm) {
    m_global = o.m_global;
    if (m_global == 0) {  // R6 needs the global m: one combine of the ranks' m at the start
      o.comm->epoch += 1;
      CommDev cd;
      fill_comm(cd, o.comm);
      double* d_m = c->d_scratch + 4;
      int* d_err = (int*)(c->d_scratch + 5);
      if (launch_comm_sum(cd, o.comm->epoch, (double)m, d_m, d_err, s)) return fail(JF_ECUDA);
      CK(cudaMemcpyAsync(c->h_pin, d_m, sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(c->h_pin + 1, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(stream_wait(s));
      if (*(int*)(c->h_pin + 1)) return fail(JF_ECOMM);
      m_global = (int64_t)c->h_pin[0];
    }
  }

  // trace buffer
  if (o.trace_cap > 0) {
    if (!o.trace) return fail(JF_EINVAL);
    size_t cap = (size_t)c->trace_cap * TRACE_FIELDS;
    if (int e = ensure(c->d_trace, cap, (size_t)o.trace_cap * TRACE_FIELDS, s)) return fail(e);
    c->trace_cap = (int)(cap / TRACE_FIELDS);
  }

  // ---- device state
  FitState& h = *c->h_state;
  memset(&h, 0, sizeof(h));
  h.n = n;
  h.bounded = bounded ? 1 : 0;
  h.jacmode = (o.x_scale_mode == JF_XSCALE_JAC) ? 1 : 0;
  h.max_nfev = o.max_nfev > 0 ? o.max_nfev : 100 * n;
  h.policy = o.policy;
  h.trace_cap = o.trace_cap > 0 ? o.trace_cap : 0;
  h.trace = c->d_trace;
  h.m_global = m_global;
  h.ftol = o.ftol;
  h.xtol = o.xtol;
  h.gtol = o.gtol;
  for (int j = 0; j < NMAX; ++j) {
    h.lb[j] = j < n ? L[j] : 0.0;
    h.ub[j] = j < n ? U[j] : 0.0;
    h.xs_inv[j] = j < n ? XS[j] : 1.0;
    h.x[j] = j < n ? X0[j] : 0.0;
    h.x_eval[j] = h.x[j];
  }
  // TSQR or AUTO (decided on the device after the first pass) need the
  // preconditioned-pass node in the graph
  const bool qr = (o.solver == JF_SOLVE_TSQR || o.solver == JF_SOLVE_AUTO);
  h.qr_mode = (o.solver == JF_SOLVE_TSQR) ? 1 : (o.solver == JF_SOLVE_AUTO ? 2 : 0);
  h.auto_mode = (o.solver == JF_SOLVE_AUTO) ? 1 : 0;
  h.kappa2_gn = 0.0;
  h.qr = c->d_qr;
  h.prec = c->d_qr->prec;
  if (n == 7) {  // the first J-pass's prologue (the solver step writes the later ones)
    gauss2d_prologue(h.x_eval, h.pre);
    h.has_pre = 1;
  } else if (n == 13) {
    gauss2d_x2_prologue(h.x_eval, h.pre);
    h.has_pre = 1;
  }
  h.phase = PH_INIT_J;
  h.status = STATUS_NONE;
  h.cont = 1;
  h.comm_epoch = o.comm ? o.comm->epoch : 0ull;
  PassArgs a;
  memset(&a, 0, sizeof(a));  // padding too: compared bytewise with the last upload
  fill_args(a, sg, m, o);
  a.epilogue = EPI_FIT;
  a.no_chain = 0;
  a.dbg = nullptr;
  a.partials = c->d_partials;
  a.ticket = c->d_ticket;
  a.out = c->d_out;
  if (o.comm) {
    a.use_comm = 1;
    fill_comm(a.comm, o.comm);
  }
  // speculative one-GPU fits of the n = 7 moment J-pass: the solver step runs
  // in the pass kernel's last block (graph body: passes only).  Sharded fits
  // keep the solver kernel: a pass's last block already waits on its peers in
  // the cross-rank combine.
  const bool fused = k.fused && o.policy == JF_POLICY_SPECULATIVE && !o.comm;
  a.fused = fused ? 1 : 0;
  JF_HSTAMP(0);
  auto t0 = std::chrono::steady_clock::now();
  const int n64_est = 10 + 8 * n + (n + 1) * (n + 2) / 2;
  constexpr double small_budget = 1.0e6;  // fp64 operations of one pass that one block absorbs
  const bool small = !o.comm && o.policy == JF_POLICY_SPECULATIVE && kk.small &&
                     (double)mg * n64_est <= small_budget;
  if (small || !o.use_graph)  // (the fit graph copies the state in and out itself)
    CK(cudaMemcpyAsync(c->d_state, &h, FITSTATE_UPLOAD, cudaMemcpyHostToDevice, s));  // (not the device-written bulk)
  JF_HSTAMP(1);
  if (!c->h_args_valid || memcmp(c->h_args, &a, sizeof(a)) != 0) {  // a repeated fit skips the copy
    *c->h_args = a;
    c->h_args_valid = true;
    CK(cudaMemcpyAsync(c->d_args, c->h_args, sizeof(a), cudaMemcpyHostToDevice, s));
  }
  int launches = 0;
  // small m: the whole fit in one single-block kernel (state in shared memory)
  if (small) {
    SmallFitFn f = sg.wsig ? kk.smallw : kk.small;
    f<<<1, 256, 0, s>>>(c->d_args, c->d_state);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h, c->d_state, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(stream_wait(s));
  } else if (o.use_graph) {
    GraphKey key{(const void*)k.j, o.policy, k.jgrid, k.rgrid, (qr ? 1 : 0) | (fused ? 2 : 0)};
    auto it = c->graphs.find(key);
    cudaGraphExec_t ge;
    if (it == c->graphs.end()) {
      r = build_graph(*c, k, o.policy, qr, fused, &ge);
      if (r) return fail(r);
      c->graphs[key] = ge;
    } else {
      ge = it->second;
      out->graph_reused = 1;
    }
    nvtxRangePushA("fit graph (passes + solver steps on the device)");
    JF_HSTAMP(2);
    CK(cudaGraphLaunch(ge, s));  // (state in, passes + solver steps, state out)
    JF_HSTAMP(3);
    JF_HSTAMP(4);
    const cudaError_t we = stream_wait(s);
    JF_HSTAMP(5);
    nvtxRangePop();
    CK(we);
  } else {
    const int cap = 4 * h.max_nfev + 8;
    for (int iter = 0; iter < cap; ++iter) {
      const bool jac = (o.policy == JF_POLICY_CONSERVATIVE) ? (h.phase != PH_TRIAL_R) : true;
      {
        NvtxRange nv3(jac ? "J-pass" : "r-pass");
        r = launch_pass(k, jac, s, c->d_args, c->d_state, g_zero_args);  // J kernels also run PH_QR2
      }
      if (r) return fail(r);
      if (!fused) {
        NvtxRange nv3("solver step");
        if (launch_solver(c->d_state, c->d_out, s)) return fail(JF_ECUDA);
      }
      CK(cudaMemcpyAsync(&h, c->d_state, sizeof(h), cudaMemcpyDeviceToHost, s));
      CK(stream_wait(s));
      if (!h.cont) break;
    }
  }
  out->t_solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  launches = h.kernels;
  if (o.comm) o.comm->epoch = h.comm_epoch;

  // ---- result
  out->kernel_launches = launches;
  out->t_epilogue_s = h.epi_ns * 1e-9;
  for (int q = 0; q < 8; ++q) out->epilogue_cycles[q] = (double)h.prof[q];
  out->timeline_len = h.tl_n < 64 ? h.tl_n : 64;
  for (int q = 0; q < out->timeline_len; ++q) out->timeline_ns[q] = (double)(h.tl[q] - h.tl[0]);
  out->nfev = h.nfev;
  out->njev = h.njev;
  out->nit = h.nit;
  out->cost = h.cost;
  out->optimality = h.gnorm;
  for (int j = 0; j < n; ++j) {
    out->x[j] = h.x[j];
    out->grad[j] = h.g[j];
    for (int q = 0; q < n; ++q) {
      out->gram[j * n + q] = h.G[j * NMAX + q];
      out->pcov[j * n + q] = h.pcov[j * NMAX + q];
    }
  }
  if (bounded) active_mask_host(h.x, L, U, n, o.xtol, out->active_mask);
  out->trace_len = h.trace_len < o.trace_cap ? h.trace_len : o.trace_cap;
  if (o.trace_cap > 0 && out->trace_len > 0)
  {
    CK(cudaMemcpyAsync(o.trace, c->d_trace, sizeof(double) * TRACE_FIELDS * out->trace_len, cudaMemcpyDeviceToHost, s));
    CK(stream_wait(s));
  }
  if (h.error) return fail(h.error);
  if (h.cont) return fail(JF_ECUDA);  // loop did not terminate
  out->status = h.status;
#if JF_DEV
  JF_HSTAMP(6);
  fprintf(stderr, "fit host us: setup %.1f h2d %.1f ->launch %.1f launch %.1f d2h-enq %.1f wait %.1f results %.1f\n", hd[0],
          hd[1] - hd[0], hd[2] - hd[1], hd[3] - hd[2], hd[4] - hd[3], hd[5] - hd[4], hd[6] - hd[5]);
#endif
  return h.status;
}

int32_t jf_curve_fit(int32_t model, const double* y, const double* z, int64_t m, const double* p0, int32_t n,
                     const double* lb, const double* ub, const jf_opts* opts, jf_result* out) {
  if (!out) return JF_EINVAL;
  memset(out, 0, sizeof(*out));
  const int32_t r = fit_impl(model, y, z, m, p0, n, lb, ub, opts, out);
  if (r < 0) out->status = r;
  return r;
}

// ------------------------------------------------- batched many small fits
int32_t jf_curve_fit_batch(int32_t model, const double* y, const double* z, int64_t m, int64_t nfits,
                           const double* p0, int32_t n, const double* lb, const double* ub, const jf_opts* opts,
                           jf_batch_result* out) {
  static_assert(sizeof(jf_batch_result) == sizeof(BatchResult), "jf_batch_result layout");
  NvtxRange nv("jf_curve_fit_batch");
  jf_opts o;
  if (opts) o = *opts;
  else jf_opts_default(&o);
  const int d = model_d(model);
  if (model_n(model) < 0 || n != model_n(model) || !z || !out || m < 1 || nfits < 1 || o.comm) return JF_EINVAL;
  if (o.x_scale_mode < 0 || o.x_scale_mode > 2 || o.solver < 0 || o.solver > 2) return JF_EINVAL;
  double L[NMAX], U[NMAX], XS[NMAX];
  bool bounded = false;
  for (int j = 0; j < n; ++j) {
    L[j] = lb ? lb[j] : -INFINITY;
    U[j] = ub ? ub[j] : INFINITY;
    if (std::isnan(L[j]) || std::isnan(U[j]) || !(L[j] < U[j])) return JF_EINVAL;
    if (std::isfinite(L[j]) || std::isfinite(U[j])) bounded = true;
    XS[j] = 1.0;
  }
  if (o.x_scale_mode == JF_XSCALE_ARRAY) {
    if (!o.x_scale) return JF_EINVAL;
    for (int j = 0; j < n; ++j) {
      if (!std::isfinite(o.x_scale[j]) || !(o.x_scale[j] > 0)) return JF_EINVAL;
      XS[j] = 1.0 / o.x_scale[j];
    }
  }
  int coord = COORD_EXPLICIT;
  if (!y) {
    if (d == 2) {
      if (o.grid_w < 1 || o.grid_h < 1 || o.grid_w * o.grid_h != m) return JF_EINVAL;
      coord = COORD_GRID;
    } else {
      if (!std::isfinite(o.t0) || !std::isfinite(o.dt)) return JF_EINVAL;
      coord = COORD_IMPLICIT_T;
    }
  }
  const bool shared_y = (o.flags & JF_FLAG_BATCH_SHARED_Y) != 0;
  Kernels kk = get_kernels(model, coord);
  BatchFn f = o.sigma ? kk.batchw : kk.batch;
  if (!f) return JF_EINVAL;
  Ctx* c;
  std::unique_lock<std::mutex> lk;
  cudaStream_t s;
  int r = acquire(o, c, lk, s);
  if (r) return r;
  StreamOrder order;
  if ((r = order.begin(c, s))) return r;
  if (order.cap) return JF_EINVAL;
  // ---- data in HBM
  const size_t nz = (size_t)nfits * m;
  const size_t ny = (coord == COORD_EXPLICIT) ? (size_t)d * m * (shared_y ? 1 : nfits) : 0;
  const size_t nw = o.sigma ? nz : 0;
  const size_t np0 = p0 ? (size_t)nfits * n : 0;
  BatchArgs ba;
  memset(&ba, 0, sizeof(ba));
  const double *zd = z, *yd = y, *wd = o.sigma, *pd = p0;
  const size_t need = (o.inputs_on_device ? 0 : nz + ny) + nw + np0;
  if (int e = ensure(c->d_in, c->in_cap, need, s)) return e;
  double* q = c->d_in;
  if (!o.inputs_on_device) {
    CK(cudaMemcpyAsync(q, z, sizeof(double) * nz, cudaMemcpyHostToDevice, s));
    zd = q;
    q += nz;
    if (ny) {
      CK(cudaMemcpyAsync(q, y, sizeof(double) * ny, cudaMemcpyHostToDevice, s));
      yd = q;
      q += ny;
    }
  }
  if (nw) {  // 1 / sigma
    CK(cudaMemcpyAsync(q, o.sigma, sizeof(double) * nw, o.inputs_on_device ? cudaMemcpyDeviceToDevice
                                                                           : cudaMemcpyHostToDevice, s));
    inv_kernel<<<c->nsm * 4, 256, 0, s>>>(q, (int64_t)nw);
    CK(cudaGetLastError());
    wd = q;
    q += nw;
  }
  if (np0) {  // p0 always from the host
    CK(cudaMemcpyAsync(q, p0, sizeof(double) * np0, cudaMemcpyHostToDevice, s));
    pd = q;
    q += np0;
  }
  // ---- the shared configuration (a FitState template)
  if (!c->d_tmpl) CK(cudaMalloc(&c->d_tmpl, sizeof(FitState)));
  FitState& h = *c->h_state;
  memset(&h, 0, sizeof(h));
  h.n = n;
  h.bounded = bounded ? 1 : 0;
  h.jacmode = (o.x_scale_mode == JF_XSCALE_JAC) ? 1 : 0;
  h.max_nfev = o.max_nfev > 0 ? o.max_nfev : 100 * n;
  h.policy = JF_POLICY_SPECULATIVE;
  h.m_global = m;
  h.ftol = o.ftol;
  h.xtol = o.xtol;
  h.gtol = o.gtol;
  for (int j = 0; j < NMAX; ++j) {
    h.lb[j] = j < n ? L[j] : 0.0;
    h.ub[j] = j < n ? U[j] : 0.0;
    h.xs_inv[j] = j < n ? XS[j] : 1.0;
  }
  h.qr_mode = (o.solver == JF_SOLVE_TSQR) ? 1 : (o.solver == JF_SOLVE_AUTO ? 2 : 0);
  h.auto_mode = (o.solver == JF_SOLVE_AUTO) ? 1 : 0;
  if (n == 7) {  // the first J-pass's prologue (the solver step writes the later ones)
    gauss2d_prologue(h.x_eval, h.pre);
    h.has_pre = 1;
  } else if (n == 13) {
    gauss2d_x2_prologue(h.x_eval, h.pre);
    h.has_pre = 1;
  }
  h.phase = PH_INIT_J;
  h.status = STATUS_NONE;
  h.cont = 1;
  CK(cudaMemcpyAsync(c->d_tmpl, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  // ---- launch: one warp per fit, persistent blocks
  static std::mutex occ_mu;
  static std::map<std::pair<int, const void*>, int> occ_cache;
  int occ = 1;
  {
    std::lock_guard<std::mutex> g(occ_mu);
    auto key = std::make_pair(c->dev, (const void*)f);
    auto it = occ_cache.find(key);
    if (it == occ_cache.end()) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 32, 0) != cudaSuccess || occ < 1) occ = 1;
      occ_cache[key] = occ;
    } else {
      occ = it->second;
    }
  }
  const int grid = (int)std::min<int64_t>(nfits, (int64_t)c->nsm * occ);
  if (c->qr_batch_cap < grid) {
    if (c->d_qr_batch) CK(cudaFreeAsync(c->d_qr_batch, s));
    CK(cudaMallocAsync((void**)&c->d_qr_batch, sizeof(QRState) * grid, s));
    c->qr_batch_cap = grid;
  }
  if (c->bout_cap < (size_t)nfits) {
    if (c->d_bout) CK(cudaFreeAsync(c->d_bout, s));
    CK(cudaMallocAsync((void**)&c->d_bout, sizeof(BatchResult) * nfits, s));
    c->bout_cap = nfits;
  }
  Staged sg;
  sg.z = zd;
  sg.coord = coord;
  if (coord == COORD_EXPLICIT) {
    sg.y0 = yd;
    sg.y1 = (d == 2) ? yd + m : nullptr;
  }
  sg.wsig = wd;
  fill_args(ba.base, sg, m, o);
  ba.base.epilogue = EPI_NONE;
  ba.nfits = nfits;
  ba.z_stride = m;
  ba.y_stride = (coord == COORD_EXPLICIT && !shared_y) ? (int64_t)d * m : 0;
  ba.p0 = pd;
  ba.tmpl = c->d_tmpl;
  ba.qr = c->d_qr_batch;
  ba.out = c->d_bout;
  f<<<grid, 32, 0, s>>>(ba);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, c->d_bout, sizeof(BatchResult) * nfits, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

// ----------------------------------------------------- subproblem test hook
}  // extern "C"


extern "C" int32_t jf_trust_region_step(const double* hatG, const double* hatg, int32_t n, int64_t m, double Delta,
                                        double alpha_in, const jf_opts* opts, double* p, double* alpha_out,
                                        int32_t* n_iter) {
  jf_opts o;
  if (opts) o = *opts;
  else jf_opts_default(&o);
  if (!hatG || !hatg || !p || n < 1 || n > NMAX || !(Delta > 0)) return JF_EINVAL;
  Ctx* c;
  std::unique_lock<std::mutex> lk;
  cudaStream_t s;
  int r = acquire(o, c, lk, s);
  if (r) return r;
  double* d = c->d_scratch + 8;
  double* dG = d;
  double* dg = d + n * n;
  double* dout = dg + n;
  CK(cudaMemcpyAsync(dG, hatG, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dg, hatg, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (launch_tr_step(dG, dg, n, m, Delta, alpha_in, dout, 0, s)) return JF_ECUDA;
  double hout[2 * NMAX + 2];
  CK(cudaMemcpyAsync(hout, dout, sizeof(hout), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int j = 0; j < n; ++j) p[j] = hout[j];
  if (alpha_out) *alpha_out = hout[2 * NMAX];
  if (n_iter) *n_iter = (int32_t)hout[2 * NMAX + 1];
  return 0;
}

extern "C" int32_t jf_select_step(const double* hatB, const double* hatg, const double* x, const double* lb,
                                  const double* ub, const double* d, const double* p_h, int32_t n, double Delta,
                                  double theta, const jf_opts* opts, double* step, double* step_h, double* pred,
                                  int32_t* branch) {
  jf_opts o;
  if (opts) o = *opts;
  else jf_opts_default(&o);
  if (!hatB || !hatg || !x || !lb || !ub || !d || !p_h || !step || n < 1 || n > NMAX || !(Delta > 0)) return JF_EINVAL;
  Ctx* c;
  std::unique_lock<std::mutex> lk;
  cudaStream_t s;
  int r = acquire(o, c, lk, s);
  if (r) return r;
  StreamOrder order;
  if ((r = order.begin(c, s))) return r;
  double hin[NMAX * NMAX + 6 * NMAX];
  memcpy(hin, hatB, sizeof(double) * n * n);
  const double* src[6] = {hatg, x, lb, ub, d, p_h};
  for (int q = 0; q < 6; ++q) memcpy(hin + n * n + q * n, src[q], sizeof(double) * n);
  double* din = c->d_scratch + 8;
  double* dout = din + NMAX * NMAX + 6 * NMAX;
  CK(cudaMemcpyAsync(din, hin, sizeof(double) * (n * n + 6 * n), cudaMemcpyHostToDevice, s));
  if (launch_select_step(din, n, Delta, theta, dout, s)) return JF_ECUDA;
  double hout[2 * NMAX + 2];
  CK(cudaMemcpyAsync(hout, dout, sizeof(hout), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int j = 0; j < n; ++j) {
    step[j] = hout[j];
    if (step_h) step_h[j] = hout[NMAX + j];
  }
  if (pred) *pred = hout[2 * NMAX];
  if (branch) *branch = (int32_t)hout[2 * NMAX + 1];
  return 0;
}

// ============================================================ multi-GPU comm
// Mailbox-based cross-rank combine (jf.h "Multi-GPU").  Each rank allocates
// one mailbox in its own HBM; peers map it through CUDA IPC and write into it
// over NVLink from inside the pass kernel (jf_pass.cuh comm_combine).
namespace {
struct HandleBlob {
  uint32_t magic;
  int32_t rank, nranks, device;
  cudaIpcMemHandle_t h;
};
constexpr uint32_t kMagic = 0x4a464232u;  // "JFB2"
}  // namespace

extern "C" {

int32_t jf_comm_create(int32_t rank, int32_t nranks, int32_t device, jf_comm** comm) {
  if (!comm || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) return JF_EINVAL;
  *comm = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return JF_ECUDA;
  jf_comm* c = new jf_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  if (cudaMalloc(&c->mbox, mbox_bytes(nranks)) != cudaSuccess) {
    delete c;
    return JF_ENOMEM;
  }
  if (cudaMemset(c->mbox, 0, mbox_bytes(nranks)) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
    cudaFree(c->mbox);
    delete c;
    return JF_ECUDA;
  }
  c->peer[rank] = c->mbox;
  *comm = c;
  return 0;
}

int32_t jf_comm_export(const jf_comm* comm, uint8_t handle[JF_COMM_HANDLE_BYTES]) {
  if (!comm || !handle || comm->local) return JF_EINVAL;
  HandleBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagic;
  b.rank = comm->rank;
  b.nranks = comm->nranks;
  b.device = comm->device;
  if (cudaSetDevice(comm->device) != cudaSuccess) return JF_ECUDA;
  if (cudaIpcGetMemHandle(&b.h, comm->mbox) != cudaSuccess) return JF_ECOMM;
  memset(handle, 0, JF_COMM_HANDLE_BYTES);
  memcpy(handle, &b, sizeof(b));
  return 0;
}

int32_t jf_comm_connect(jf_comm* comm, const uint8_t* all) {
  if (!comm || !all || comm->local) return JF_EINVAL;
  if (cudaSetDevice(comm->device) != cudaSuccess) return JF_ECUDA;
  for (int p = 0; p < comm->nranks; ++p) {
    HandleBlob b;
    memcpy(&b, all + (size_t)p * JF_COMM_HANDLE_BYTES, sizeof(b));
    if (b.magic != kMagic || b.rank != p || b.nranks != comm->nranks) return JF_EINVAL;
    if (p == comm->rank) continue;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, comm->device, b.device) == cudaSuccess && can) {
      cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return JF_ECOMM;
      cudaGetLastError();
    }
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, b.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return JF_ECOMM;
    comm->peer[p] = ptr;
    comm->opened[p] = true;
  }
  return 0;
}

int32_t jf_comm_create_local(int32_t nranks, int32_t device, jf_comm** comms) {
  if (!comms || nranks < 1 || nranks > 8) return JF_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return JF_ECUDA;
  std::vector<jf_comm*> cs;
  for (int r = 0; r < nranks; ++r) {
    jf_comm* c = nullptr;
    int e = jf_comm_create(r, nranks, device, &c);
    if (e) {
      for (auto* q : cs) jf_comm_destroy(q);
      return e;
    }
    c->local = true;
    cs.push_back(c);
  }
  for (int r = 0; r < nranks; ++r)
    for (int p = 0; p < nranks; ++p) cs[r]->peer[p] = cs[p]->mbox;
  // initialise the emulated ranks' contexts now: a context created while a
  // peer's pass kernel spins on its mailbox could otherwise wait on it
  for (int r = 0; r < nranks; ++r) {
    Ctx& c = g_ctx[64 + device * 8 + r];
    std::lock_guard<std::mutex> g(c.mu);
    if (int e = ctx_init(c, device)) {
      for (auto* q : cs) jf_comm_destroy(q);
      return e;
    }
  }
  for (int r = 0; r < nranks; ++r) comms[r] = cs[r];
  return 0;
}

int32_t jf_comm_set_timeout(jf_comm* comm, int32_t timeout_ms) {
  if (!comm || timeout_ms < 1) return JF_EINVAL;
  comm->timeout_ns = (unsigned long long)timeout_ms * 1000000ull;
  return 0;
}

int32_t jf_comm_bench(jf_comm* comm, double v, int32_t reps, double* sum, double* us) {
  if (!comm || reps < 1) return JF_EINVAL;
  jf_opts o;
  jf_opts_default(&o);
  o.device = comm->device;
  o.comm = comm;
  Ctx* c;
  std::unique_lock<std::mutex> lk;
  cudaStream_t s;
  int r = acquire(o, c, lk, s);
  if (r) return r;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  double* d_v = c->d_scratch + 4;
  int* d_err = (int*)(c->d_scratch + 5);
  CommDev cd;
  fill_comm(cd, comm);
  comm->epoch += 1;  // one warm-up combine
  if (launch_comm_sum(cd, comm->epoch, v, d_v, d_err, s)) return JF_ECUDA;
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < reps; ++i) {
    comm->epoch += 1;
    if (launch_comm_sum(cd, comm->epoch, v, d_v, d_err, s)) return JF_ECUDA;
  }
  CK(cudaEventRecord(e1, s));
  CK(cudaMemcpyAsync(c->h_pin, d_v, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(c->h_pin + 1, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const double hv = c->h_pin[0];
  const int herr = *(int*)(c->h_pin + 1);
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (herr) return JF_ECOMM;
  if (sum) *sum = hv;
  if (us) *us = 1e3 * ms / reps;
  return 0;
}

int32_t jf_graph_cache_clear(int32_t device) {
  if (device < 0 || device >= 64) return JF_EINVAL;
  Ctx& c = g_ctx[device];
  std::lock_guard<std::mutex> g(c.mu);
  if (!c.ready) return 0;
  if (cudaSetDevice(device) != cudaSuccess) return JF_ECUDA;
  if (c.done_stream) cudaEventSynchronize(c.done);
  for (auto& kv : c.graphs) cudaGraphExecDestroy(kv.second);
  c.graphs.clear();
  return 0;
}

int32_t jf_comm_destroy(jf_comm* comm) {
  if (!comm) return JF_EINVAL;
  cudaSetDevice(comm->device);
  cudaDeviceSynchronize();
  for (int p = 0; p < comm->nranks; ++p)
    if (comm->opened[p]) cudaIpcCloseMemHandle(comm->peer[p]);
  if (comm->mbox) cudaFree(comm->mbox);
  delete comm;
  return 0;
}

}  // extern "C"

"""Thin Python API over the C ABI (include/jf.h) — argument marshalling only.

Names follow jf.h: curve_fit (jf_curve_fit), jpass (jf_pass), residual_pass
(jf_residual_pass), pass_device (jf_pass_device), trust_region_step
(jf_trust_region_step), Comm (jf_comm_*).  Arrays may be numpy (host
memory: the library copies them to HBM) or CUDA torch tensors (device
memory: read in place).  No computation happens here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class JFError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = L.load().jf_strerror(code).decode()
        super().__init__(f"{where}: {msg} ({code})")


def _model_id(model) -> int:
    if isinstance(model, str):
        return L.MODEL_IDS[model]
    return int(model)


def nparams(model) -> int:
    return L.load().jf_model_nparams(_model_id(model))


def _dptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _is_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _as_host(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class _Data:
    """Holds the (y, z, sigma) buffers alive and resolves their pointers."""

    def keep_alive(self, stream_ptr):
        """Tell torch's caching allocator that converted copies are in use on
        the library's stream until the work enqueued there completes."""
        if not self.on_device or not self._tmp:
            return
        import torch
        s = torch.cuda.ExternalStream(stream_ptr) if stream_ptr else torch.cuda.current_stream()
        for t in self._tmp:
            t.record_stream(s)

    def __init__(self, y, z, sigma):
        self.on_device = _is_cuda(z)
        if self.on_device:
            import torch
            for t in (y, sigma):
                if t is not None and not _is_cuda(t):
                    raise ValueError("z is a CUDA tensor: y and sigma must be CUDA tensors too")
            self.z = z.contiguous().to(torch.float64)
            self.y = None if y is None else y.contiguous().to(torch.float64)
            self.sigma = None if sigma is None else sigma.contiguous().to(torch.float64)
            self.zp = self.z.data_ptr()
            self.yp = None if self.y is None else self.y.data_ptr()
            self.sp = None if self.sigma is None else self.sigma.data_ptr()
            self.m = int(self.z.numel())
            self._tmp = [t for t, u in ((self.z, z), (self.y, y), (self.sigma, sigma))
                         if t is not None and t.data_ptr() != u.data_ptr()]
        else:
            self.z = _as_host(z)
            self.y = None if y is None else _as_host(y)
            self.sigma = None if sigma is None else _as_host(sigma)
            self.zp = self.z.ctypes.data
            self.yp = None if self.y is None else self.y.ctypes.data
            self.sp = None if self.sigma is None else self.sigma.ctypes.data
            self.m = int(self.z.size)


def _default_stream(on_device, stream):
    """CUDA inputs: run on torch's current stream unless told otherwise, so
    the library's work is ordered after the work that produced the inputs."""
    if stream is None and on_device:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream


def make_opts(*, grid=None, t0=0.0, dt=1.0, index0=0, sigma_ptr=None, on_device=False, device=0,
              stream=None, ftol=1e-8, xtol=1e-8, gtol=1e-8, max_nfev=0, x_scale="jac",
              policy="speculative", use_graph=True, comm=None, m_global=0, solver="auto", capacity=0,
              alt_coords=False):
    lib = L.load()
    o = L.jf_opts()
    lib.jf_opts_default(C.byref(o))
    o.ftol, o.xtol, o.gtol = ftol, xtol, gtol
    o.max_nfev = int(max_nfev or 0)
    keep = []
    if isinstance(x_scale, str):
        o.x_scale_mode = {"jac": L.XSCALE_JAC, "ones": L.XSCALE_ONES}[x_scale]
    else:
        xs = _as_host(x_scale)
        keep.append(xs)
        o.x_scale_mode = L.XSCALE_ARRAY
        o.x_scale = _dptr(xs)
    o.policy = {"speculative": L.POLICY_SPECULATIVE, "conservative": L.POLICY_CONSERVATIVE}[policy]
    o.solver = {"auto": L.SOLVE_AUTO, "gram": L.SOLVE_GRAM, "tsqr": L.SOLVE_TSQR}[solver]
    if grid is not None:
        o.grid_w, o.grid_h = int(grid[0]), int(grid[1])
        o.grid_row0 = int(grid[2]) if len(grid) > 2 else 0
    o.t0, o.dt, o.index0 = float(t0), float(dt), int(index0)
    o.sigma = sigma_ptr
    o.device = int(device)
    o.inputs_on_device = 1 if on_device else 0
    o.capacity = int(capacity)
    o.flags = L.FLAG_ALT_COORDS if alt_coords else 0
    stream = _default_stream(on_device, stream)
    if stream is not None:
        o.stream = stream if isinstance(stream, int) else int(getattr(stream, "cuda_stream", stream))
    o.use_graph = 1 if use_graph else 0
    if comm is not None:
        o.comm = comm.handle
        o.m_global = int(m_global)
    return o, keep


class FitResult:
    """jf_result as Python values.  The arrays are built from the C struct on
    first access (marshalling only; a fit's wall time then does not pay for
    arrays the caller never reads)."""

    _ARRAYS = {"x": 1, "grad": 1, "gram": 2, "pcov": 2}
    _SCALARS = ("cost", "optimality", "status", "nfev", "njev", "nit", "kernel_launches", "graph_reused",
                "t_upload_s", "t_solve_s", "t_epilogue_s")

    def __init__(self, res, n, trace=None):
        self._res = res
        self._n = n
        self._cache = {}
        self.trace = trace if trace is not None else np.zeros((0, L.JF_TRACE_FIELDS))

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        cache = self._cache
        if name in cache:
            return cache[name]
        res, n = self._res, self._n
        if name in self._SCALARS:
            v = getattr(res, name)
        elif name in self._ARRAYS:
            k = n if self._ARRAYS[name] == 1 else n * n
            v = np.frombuffer(getattr(res, name), dtype=np.float64, count=k).copy()
            if self._ARRAYS[name] == 2:
                v = v.reshape(n, n)
        elif name == "active_mask":
            v = np.frombuffer(res.active_mask, dtype=np.int8, count=n).astype(np.int64)
        elif name == "epilogue_cycles":
            v = np.frombuffer(res.epilogue_cycles, dtype=np.float64, count=8).copy()
        elif name == "timeline_ns":
            v = np.frombuffer(res.timeline_ns, dtype=np.float64, count=res.timeline_len).copy()
        else:
            raise AttributeError(name)
        cache[name] = v
        return v

    def __repr__(self):
        return (f"FitResult(status={self.status}, nfev={self.nfev}, njev={self.njev}, nit={self.nit}, "
                f"cost={self.cost!r}, x={self.x!r})")


def curve_fit(model, z, y=None, *, grid=None, p0=None, lb=None, ub=None, sigma=None, trace_cap=0,
              **kw) -> FitResult:
    """jf_curve_fit: minimise 1/2 sum (h(y_i; x) - z_i)^2 by TRF."""
    lib = L.load()
    mid = _model_id(model)
    n = lib.jf_model_nparams(mid)
    data = _Data(y, z, sigma)
    opts, keep = make_opts(grid=grid, sigma_ptr=data.sp, on_device=data.on_device, **kw)
    tr = None
    if trace_cap > 0:
        tr = np.zeros((trace_cap, L.JF_TRACE_FIELDS))
        opts.trace_cap = trace_cap
        opts.trace = _dptr(tr)
    p0a = None if p0 is None else _as_host(p0)
    lba = None if lb is None else _as_host(lb)
    uba = None if ub is None else _as_host(ub)
    res = L.jf_result()
    rc = lib.jf_curve_fit(mid, data.yp, data.zp, data.m, None if p0a is None else p0a.ctypes.data, n,
                          None if lba is None else lba.ctypes.data, None if uba is None else uba.ctypes.data,
                          C.byref(opts), C.byref(res))
    if rc < 0:
        raise JFError(rc, "jf_curve_fit")
    out = FitResult(res, n)
    if tr is not None:
        out.trace = tr[: res.trace_len].copy()
    return out


@dataclass
class BatchResult:
    x: np.ndarray          # (nfits, n)
    cost: np.ndarray
    optimality: np.ndarray
    status: np.ndarray
    nfev: np.ndarray
    njev: np.ndarray
    nit: np.ndarray


def curve_fit_batch(model, z, y=None, *, grid=None, p0=None, lb=None, ub=None, sigma=None, shared_y=False,
                    **kw) -> BatchResult:
    """jf_curve_fit_batch: one TRF fit per row of z (nfits x m) in one launch."""
    lib = L.load()
    mid = _model_id(model)
    n = lib.jf_model_nparams(mid)
    nfits, m = int(z.shape[0]), int(z.shape[1])
    data = _Data(y, z.reshape(-1) if not _is_cuda(z) else z.reshape(-1), sigma)
    opts, keep = make_opts(grid=grid, sigma_ptr=data.sp, on_device=data.on_device, **kw)
    if shared_y:
        opts.flags |= L.FLAG_BATCH_SHARED_Y
    p0a = None if p0 is None else _as_host(p0).reshape(nfits, n)
    lba = None if lb is None else _as_host(lb)
    uba = None if ub is None else _as_host(ub)
    out = (L.jf_batch_result * nfits)()
    rc = lib.jf_curve_fit_batch(mid, data.yp, data.zp, m, nfits, None if p0a is None else p0a.ctypes.data, n,
                                None if lba is None else lba.ctypes.data, None if uba is None else uba.ctypes.data,
                                C.byref(opts), out)
    if rc < 0:
        raise JFError(rc, "jf_curve_fit_batch")
    rec = np.frombuffer(out, dtype=np.dtype([("x", np.float64, L.JF_MAX_N), ("cost", np.float64),
                                             ("optimality", np.float64), ("status", np.int32),
                                             ("nfev", np.int32), ("njev", np.int32), ("nit", np.int32)]))
    return BatchResult(x=rec["x"][:, :n].copy(), cost=rec["cost"].copy(), optimality=rec["optimality"].copy(),
                       status=rec["status"].copy(), nfev=rec["nfev"].copy(), njev=rec["njev"].copy(),
                       nit=rec["nit"].copy())


def jpass(model, z, x, y=None, *, grid=None, sigma=None, **kw):
    """jf_pass: (cost, g, G, nonfinite) at x (Eq. 2, 4, 5)."""
    lib = L.load()
    mid = _model_id(model)
    n = lib.jf_model_nparams(mid)
    data = _Data(y, z, sigma)
    opts, keep = make_opts(grid=grid, sigma_ptr=data.sp, on_device=data.on_device, **kw)
    xa = _as_host(x)
    cost = C.c_double()
    g = np.zeros(n)
    G = np.zeros(n * n)
    bad = C.c_int32()
    rc = lib.jf_pass(mid, data.yp, data.zp, data.m, _dptr(xa), n, C.byref(opts), C.byref(cost), _dptr(g),
                     _dptr(G), C.byref(bad))
    if rc < 0:
        raise JFError(rc, "jf_pass")
    return cost.value, g, G.reshape(n, n), bad.value


def residual_pass(model, z, x, y=None, *, grid=None, sigma=None, **kw):
    """jf_residual_pass: (cost, nonfinite) at x."""
    lib = L.load()
    mid = _model_id(model)
    n = lib.jf_model_nparams(mid)
    data = _Data(y, z, sigma)
    opts, keep = make_opts(grid=grid, sigma_ptr=data.sp, on_device=data.on_device, **kw)
    xa = _as_host(x)
    cost = C.c_double()
    bad = C.c_int32()
    rc = lib.jf_residual_pass(mid, data.yp, data.zp, data.m, _dptr(xa), n, C.byref(opts), C.byref(cost),
                              C.byref(bad))
    if rc < 0:
        raise JFError(rc, "jf_residual_pass")
    return cost.value, bad.value


def pass_device(model, z, x_dev, kvec_dev, y=None, *, grid=None, sigma=None, residual_only=False, x_host=None,
                **kw):
    """jf_pass_device: enqueue one pass on opts.stream (all CUDA tensors).
    x_host: optional host copy of x_dev (opts.x_host: the moment J-pass then
    takes its parameter-only prologue from the call, as inside a fit)."""
    lib = L.load()
    mid = _model_id(model)
    n = lib.jf_model_nparams(mid)
    data = _Data(y, z, sigma)
    if not data.on_device:
        raise ValueError("pass_device needs CUDA tensors")
    opts, keep = make_opts(grid=grid, sigma_ptr=data.sp, on_device=True, **kw)
    if x_host is not None:
        xh = _as_host(x_host)
        if xh.size != n:
            raise ValueError("x_host must hold the n parameters")
        keep.append(xh)
        opts.x_host = _dptr(xh)
    rc = lib.jf_pass_device(mid, data.yp, data.zp, data.m, x_dev.data_ptr(), n, C.byref(opts),
                            1 if residual_only else 0, kvec_dev.data_ptr())
    if rc < 0:
        raise JFError(rc, "jf_pass_device")
    # the pass runs asynchronously: converted temporaries must outlive it
    data.keep_alive(opts.stream)


def trust_region_step(hatG, hatg, m, Delta, alpha=0.0, device=0):
    """jf_trust_region_step: the single-warp subproblem (Alg. 2 + App. B)."""
    lib = L.load()
    G = _as_host(hatG)
    g = _as_host(hatg)
    n = g.size
    p = np.zeros(n)
    a = C.c_double()
    it = C.c_int32()
    opts, _ = make_opts(device=device)
    rc = lib.jf_trust_region_step(_dptr(G), _dptr(g), n, int(m), float(Delta), float(alpha), C.byref(opts),
                                  _dptr(p), C.byref(a), C.byref(it))
    if rc < 0:
        raise JFError(rc, "jf_trust_region_step")
    return p, a.value, it.value


def select_step(hatB, hatg, x, lb, ub, d, p_h, Delta, theta, device=0):
    """jf_select_step: the device Coleman-Li step selection (R19/R20).
    Returns (step, step_h, pred, branch)."""
    lib = L.load()
    a = [_as_host(v) for v in (hatB, hatg, x, lb, ub, d, p_h)]
    n = a[1].size
    step, step_h = np.zeros(n), np.zeros(n)
    pred, br = C.c_double(), C.c_int32()
    opts, _ = make_opts(device=device)
    rc = lib.jf_select_step(*[_dptr(v) for v in a], n, float(Delta), float(theta), C.byref(opts), _dptr(step),
                            _dptr(step_h), C.byref(pred), C.byref(br))
    if rc < 0:
        raise JFError(rc, "jf_select_step")
    return step, step_h, pred.value, br.value


def graph_cache_clear(device: int = 0):
    """jf_graph_cache_clear: the next fit on `device` instantiates its graph afresh."""
    rc = L.load().jf_graph_cache_clear(int(device))
    if rc < 0:
        raise JFError(rc, "jf_graph_cache_clear")


def exchange_handles(blob: bytes, dist) -> bytes:
    """All-gather one fixed-size byte blob per rank (rank order) through a
    torch.distributed process group; returns the concatenation."""
    import torch
    n = len(blob)
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8).clone()
    if dist.get_backend() == "nccl":
        t = t.cuda()
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    res = b"".join(bytes(o.cpu().numpy().tobytes()) for o in out)
    assert len(res) == n * dist.get_world_size()
    return res


class Comm:
    """jf_comm: one rank's mailbox for the in-kernel cross-GPU combine."""

    def __init__(self, handle, lib=None):
        self.handle = handle
        self._lib = lib or L.load()

    @classmethod
    def create(cls, rank: int, nranks: int, device: int) -> "Comm":
        lib = L.load()
        h = C.c_void_p()
        rc = lib.jf_comm_create(rank, nranks, device, C.byref(h))
        if rc < 0:
            raise JFError(rc, "jf_comm_create")
        return cls(h.value, lib)

    @classmethod
    def create_local(cls, nranks: int, device: int = 0) -> list["Comm"]:
        lib = L.load()
        arr = (C.c_void_p * nranks)()
        rc = lib.jf_comm_create_local(nranks, device, arr)
        if rc < 0:
            raise JFError(rc, "jf_comm_create_local")
        return [cls(arr[i], lib) for i in range(nranks)]

    def export(self) -> bytes:
        buf = C.create_string_buffer(L.JF_COMM_HANDLE_BYTES)
        rc = self._lib.jf_comm_export(self.handle, buf)
        if rc < 0:
            raise JFError(rc, "jf_comm_export")
        return buf.raw

    def connect(self, all_handles: bytes):
        rc = self._lib.jf_comm_connect(self.handle, all_handles)
        if rc < 0:
            raise JFError(rc, "jf_comm_connect")

    @classmethod
    def from_process_group(cls, rank: int, world: int, device: int, dist=None) -> "Comm":
        """Create this rank's mailbox and connect to every peer, exchanging the
        IPC handles through torch.distributed (any backend)."""
        if dist is None:
            import torch.distributed as dist
        c = cls.create(rank, world, device)
        c.connect(exchange_handles(c.export(), dist))
        return c

    def set_timeout(self, ms: int):
        """jf_comm_set_timeout: report JF_ECOMM when a peer is missing for ms."""
        rc = self._lib.jf_comm_set_timeout(self.handle, int(ms))
        if rc < 0:
            raise JFError(rc, "jf_comm_set_timeout")

    def bench(self, v: float, reps: int = 100):
        """jf_comm_bench: (rank-ordered sum of v over the ranks, us per combine)."""
        sm, us = C.c_double(), C.c_double()
        rc = self._lib.jf_comm_bench(self.handle, float(v), int(reps), C.byref(sm), C.byref(us))
        if rc < 0:
            raise JFError(rc, "jf_comm_bench")
        return sm.value, us.value

    def destroy(self):
        if self.handle:
            self._lib.jf_comm_destroy(self.handle)
            self.handle = None

"""The C-ABI boundary's contract on the GPU (include/jf.h): fixed-capacity
graph reuse (N3, App. A), the AUTO solver along the trajectory,
passes captured into a CUDA graph, calls on different streams, the
m_global = 0 startup combine and the missing-peer timeout of the in-kernel
cross-rank combine."""
import threading

import numpy as np
import pytest

import datagen as dg
from oracle import passes as orp
from oracle import trf as otrf

jf = pytest.importorskip("paper_2208_12187_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _same_traj(res, ref):
    assert (res.status, res.nfev, res.njev, res.nit) == (ref["status"], ref["nfev"], ref["njev"], ref["nit"])
    x = ref["x"]
    assert np.all(np.abs(res.x - x) <= 1e-6 * np.maximum(np.abs(x), 1e-3 * np.max(np.abs(x))))


@pytest.mark.parametrize("model", ["gauss2d_rot", "gauss1d"])
def test_capacity_one_graph_serves_every_m(model):
    """N3: with a fixed capacity every fit of m <= capacity points replays ONE
    instantiated graph (m is read from device memory at run time, points beyond
    it are never read); each fit is bitwise identical to the same fit through a
    freshly instantiated graph and follows the oracle's trajectory."""
    if model == "gauss2d_rot":
        W, cap = 256, 256 * 256
        probs = [dg.make_gauss2d(W, H=H, seed=21) for H in (256, 201, 131)]
        kws = [dict(grid=p.grid) for p in probs]
    else:
        cap = 60_000
        probs = [dg.make_gauss1d(m, seed=22) for m in (60_000, 41_113, 25_000)]
        kws = [dict(y=p.t) for p in probs]
    jf.graph_cache_clear()
    reused = []
    for p, kw in zip(probs, kws):
        res = jf.curve_fit(p.model, p.z, p0=p.p0, capacity=cap, **kw)
        ref = otrf.fit(p.model, p.coords(), p.z, p.p0)
        _same_traj(res, ref)
        reused.append(res.graph_reused)
    assert reused == [0, 1, 1]
    again = []
    for p, kw in zip(probs, kws):
        jf.graph_cache_clear()
        fresh = jf.curve_fit(p.model, p.z, p0=p.p0, capacity=cap, **kw)
        assert fresh.graph_reused == 0
        again.append(fresh)
    for p, kw, fresh in zip(probs, kws, again):
        res = jf.curve_fit(p.model, p.z, p0=p.p0, capacity=cap, **kw)
        assert np.array_equal(res.x, fresh.x) and res.cost == fresh.cost and res.nfev == fresh.nfev
    with pytest.raises(jf.JFError) as e:  # capacity below m
        jf.curve_fit(probs[0].model, probs[0].z, p0=probs[0].p0, capacity=10, **kws[0])
    assert e.value.code == -1


@pytest.mark.parametrize("m", [20_000, 12_000])
def test_auto_switches_to_tsqr_along_the_trajectory(m):
    """AUTO starts in Gram mode (cond^2 ~ 3e2 at x0) and must take the TSQR
    path once the conditioning degrades (~3e7 at the solution): the
    trajectory stays the oracle's (SVD of J at every step).  m = 12000 runs
    the single-block whole-fit kernel, m = 20000 the graph driver."""
    t = np.arange(m) / m
    truth = np.array([1.0, 0.5, 1.0, 0.2])
    p0 = np.array([1.1, 0.5, 0.25, 0.2])
    z = dg.render("gauss1d", t, truth) + 0.01 * np.random.default_rng(7).standard_normal(m)
    ref = otrf.fit("gauss1d", t, z, p0)
    res = jf.curve_fit("gauss1d", z, y=t, p0=p0, solver="auto")
    _same_traj(res, ref)
    tsqr = jf.curve_fit("gauss1d", z, y=t, p0=p0, solver="tsqr")
    assert (tsqr.nfev, tsqr.njev) == (res.nfev, res.njev)


def test_default_solver_is_auto():
    pr = dg.make_gauss2d(200)
    a = jf.curve_fit(pr.model, pr.z, p0=pr.p0, grid=pr.grid)
    b = jf.curve_fit(pr.model, pr.z, p0=pr.p0, grid=pr.grid, solver="auto")
    assert np.array_equal(a.x, b.x) and a.nfev == b.nfev


def test_p0_none_matches_oracle_default():
    """p0 = NULL: curve_fit's default initial guess (ones; bounded: midpoint /
    bound +- 1), unbounded and bounded, against the oracle's default_p0."""
    pr = dg.make_exp_decay()
    ref = otrf.fit(pr.model, pr.t, pr.z, None)
    _same_traj(jf.curve_fit(pr.model, pr.z, y=pr.t), ref)
    lb = np.array([0.0, 0.0, -np.inf])
    ub = np.array([5.0, np.inf, 1.5])
    ref = otrf.fit(pr.model, pr.t, pr.z, None, lb, ub)
    res = jf.curve_fit(pr.model, pr.z, y=pr.t, lb=lb, ub=ub)
    _same_traj(res, ref)
    assert np.array_equal(res.active_mask, ref["active_mask"])


def test_captured_passes_keep_their_own_arguments():
    """Two pass_device calls with different parameters captured into ONE CUDA
    graph: each replayed launch uses the arguments it was captured with."""
    pr = dg.make_gauss2d(320, H=200)
    zd = torch.as_tensor(pr.z).cuda()
    x1 = torch.as_tensor(pr.p0).cuda()
    x2 = torch.as_tensor(pr.truth).cuda()
    k1 = torch.zeros(64, dtype=torch.float64, device="cuda")
    k2 = torch.zeros(64, dtype=torch.float64, device="cuda")
    r1 = torch.zeros(64, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm: kernel attributes and occupancy queries happen outside the capture
        jf.pass_device(pr.model, zd, x1, k1, grid=pr.grid, stream=s.cuda_stream)
        jf.pass_device(pr.model, zd, x1, r1, grid=pr.grid, stream=s.cuda_stream, residual_only=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        # (x_host: the prologue jpass computes, so the costs compare bitwise; the
        # precomputed prologue travels by value with each captured launch)
        jf.pass_device(pr.model, zd, x1, k1, grid=pr.grid, stream=s.cuda_stream, x_host=pr.p0)
        jf.pass_device(pr.model, zd, x2, k2, grid=pr.grid, stream=s.cuda_stream, x_host=pr.truth)
        jf.pass_device(pr.model, zd, x2, r1, grid=pr.grid, stream=s.cuda_stream, residual_only=True)
    k1.zero_()
    k2.zero_()
    jf.jpass(pr.model, pr.z, pr.p0 * 1.01, grid=pr.grid)  # other work on the library's stream in between
    g.replay()
    torch.cuda.synchronize()
    c1, _, _, _ = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    c2, _, _, _ = jf.jpass(pr.model, pr.z, pr.truth, grid=pr.grid)
    n = pr.n
    kk = (n + 1) * (n + 2) // 2
    assert k1[kk - 1].item() * 0.5 == c1 and k2[kk - 1].item() * 0.5 == c2
    assert r1[0].item() * 0.5 == pytest.approx(c2, rel=1e-12)


def test_calls_on_different_streams_are_ordered():
    """Back-to-back asynchronous passes on two streams share the context's
    buffers: the second waits for the first (no host synchronisation here)."""
    pr = dg.make_gauss2d(1024, H=700)
    zd = torch.as_tensor(pr.z).cuda()
    xs = [torch.as_tensor(pr.p0 * (1 + 0.01 * k)).cuda() for k in range(6)]
    outs = [torch.zeros(64, dtype=torch.float64, device="cuda") for _ in range(6)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for k in range(6):
        jf.pass_device(pr.model, zd, xs[k], outs[k], grid=pr.grid, stream=streams[k % 2].cuda_stream,
                       x_host=pr.p0 * (1 + 0.01 * k))  # (the prologue jpass computes: bitwise comparable)
    torch.cuda.synchronize()
    n = pr.n
    kk = (n + 1) * (n + 2) // 2
    for k in range(6):
        c, g, G, _ = jf.jpass(pr.model, pr.z, pr.p0 * (1 + 0.01 * k), grid=pr.grid)
        assert outs[k][kk - 1].item() * 0.5 == c


def _run_ranks(R, fn):
    out, err = [None] * R, [None] * R
    streams = [torch.cuda.Stream() for _ in range(R)]

    def work(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                out[r] = fn(r, streams[r])
        except Exception as e:  # pragma: no cover
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    for e in err:
        if e is not None:
            raise e
    return out


def test_m_global_zero_is_summed_over_ranks():
    """jf_opts.m_global = 0: the global m (reading R6) comes from one combine of
    the ranks' m at the start of the fit; same fit as with m_global given."""
    W, H, R = 300, 301, 3
    pr = dg.make_gauss2d(W, H=H, seed=14)
    ref = jf.curve_fit(pr.model, pr.z, p0=pr.p0, grid=pr.grid)
    comms = jf.Comm.create_local(R, 0)
    zs = [torch.as_tensor(pr.z[dg.shard_rows(H, R, r)[0] * W:dg.shard_rows(H, R, r)[1] * W]).cuda() for r in range(R)]
    torch.cuda.synchronize()
    try:
        def fn(r, s):
            r0, r1 = dg.shard_rows(H, R, r)
            return jf.curve_fit(pr.model, zs[r], p0=pr.p0, grid=(W, r1 - r0, r0), comm=comms[r], m_global=0,
                                stream=s.cuda_stream)
        outs = _run_ranks(R, fn)
        sums = _run_ranks(R, lambda r, s: comms[r].bench(float(r + 1), reps=20))
    finally:
        for c in comms:
            c.destroy()
    for o in outs:
        assert (o.status, o.nfev, o.njev, o.nit) == (ref.status, ref.nfev, ref.njev, ref.nit)
        assert np.allclose(o.x, ref.x, rtol=1e-6)
        assert np.allclose(o.pcov, ref.pcov, rtol=1e-6, atol=1e-12 * np.abs(ref.pcov).max())
    for sm, us in sums:
        assert sm == 6.0 and us > 0


def test_missing_peer_reports_ecomm():
    """A rank whose peer never arrives gets JF_ECOMM after the timeout instead
    of spinning forever (pass and fit)."""
    pr = dg.make_gauss2d(128, H=64)
    comms = jf.Comm.create_local(2, 0)
    zd = torch.as_tensor(pr.z).cuda()
    torch.cuda.synchronize()
    try:
        comms[0].set_timeout(300)
        with pytest.raises(jf.JFError) as e:
            jf.jpass(pr.model, zd, pr.p0, grid=(128, 64, 0), comm=comms[0], m_global=2 * pr.m)
        assert e.value.code == -5
        with pytest.raises(jf.JFError) as e:
            jf.curve_fit(pr.model, zd, p0=pr.p0, grid=(128, 64, 0), comm=comms[0], m_global=2 * pr.m)
        assert e.value.code == -5
    finally:
        for c in comms:
            c.destroy()

"""The multi-GPU path on ONE GPU: R virtual ranks
(jf_comm_create_local) run concurrently on separate streams; each pass kernel
pushes its K-vector into every rank's mailbox and sums them in rank order, as
on R GPUs over NVLink.  The sharded fit must match the single-rank fit of the
whole image (per-pass 1e-10 normalised; fits: identical counts, x to 1e-6)
and every rank must return the identical result."""
import threading

import numpy as np
import pytest

import datagen as dg
from oracle import passes as orp

jf = pytest.importorskip("paper_2208_12187_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _run_ranks(R, fn):
    out = [None] * R
    err = [None] * R

    streams = [torch.cuda.Stream() for _ in range(R)]

    def work(r):
        try:
            torch.cuda.set_device(0)
            s = streams[r]
            with torch.cuda.stream(s):
                out[r] = fn(r, s)
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


@pytest.mark.parametrize("R", [2, 3, 4])
def test_sharded_pass_equals_whole_image(R):
    W, H = 512, 509
    pr = dg.make_gauss2d(W, H=H, seed=12)
    comms = jf.Comm.create_local(R, 0)
    # every device allocation happens before any rank's kernel can spin on its
    # mailbox (an allocation that synchronises would wait on the spinners)
    zs = [torch.as_tensor(pr.z[dg.shard_rows(H, R, r)[0] * W:dg.shard_rows(H, R, r)[1] * W]).cuda()
          for r in range(R)]
    torch.cuda.synchronize()
    try:
        def fn(r, s):
            r0, r1 = dg.shard_rows(H, R, r)
            return jf.jpass(pr.model, zs[r], pr.p0, grid=(W, r1 - r0, r0), comm=comms[r], m_global=pr.m,
                            stream=s.cuda_stream)
        outs = _run_ranks(R, fn)
    finally:
        for c in comms:
            c.destroy()
    cr, gr, Gr, _ = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
    d = np.sqrt(np.diag(Gr))
    for c, g, G, bad in outs:
        assert bad == 0 and abs(c - cr) <= 1e-10 * cr
        assert np.all(np.abs(g - gr) <= 1e-10 * d * np.sqrt(2 * cr))
        assert np.all(np.abs(G - Gr) <= 1e-10 * np.outer(d, d))
    for o in outs[1:]:
        assert o[0] == outs[0][0] and np.array_equal(o[2], outs[0][2])


@pytest.mark.parametrize("R", [2, 4])
def test_sharded_fit_matches_single_rank(R):
    W, H = 384, 384
    pr = dg.make_gauss2d(W, H=H, seed=13)
    ref = jf.curve_fit(pr.model, pr.z, p0=pr.p0, grid=pr.grid)
    comms = jf.Comm.create_local(R, 0)
    zs = [torch.as_tensor(pr.z[dg.shard_rows(H, R, r)[0] * W:dg.shard_rows(H, R, r)[1] * W]).cuda()
          for r in range(R)]
    torch.cuda.synchronize()
    try:
        def fn(r, s):
            r0, r1 = dg.shard_rows(H, R, r)
            return jf.curve_fit(pr.model, zs[r], p0=pr.p0, grid=(W, r1 - r0, r0), comm=comms[r], m_global=pr.m,
                                stream=s.cuda_stream)
        outs = _run_ranks(R, fn)
    finally:
        for c in comms:
            c.destroy()
    for o in outs:
        assert (o.status, o.nfev, o.njev, o.nit) == (ref.status, ref.nfev, ref.njev, ref.nit)
        assert np.allclose(o.x, ref.x, rtol=1e-6)
    for o in outs[1:]:
        assert np.array_equal(o.x, outs[0].x) and o.cost == outs[0].cost


@pytest.mark.parametrize("case", range(6))
def test_sharded_random_fits_match_single_rank(case):
    """Seeded sharded fits of every model family (1D models sharded by index
    ranges with explicit t, images by row bands; 2-3 ranks): each rank returns
    the single-rank fit's counts and x, all ranks bitwise equal."""
    rng = np.random.default_rng([31, case])
    R = 2 + case % 2
    kind = case % 3
    if kind == 0:
        pr = dg.make_gauss1d(int(rng.integers(20_000, 90_000)), k=case)
    elif kind == 1:
        pr = dg.make_exp_decay(m=int(rng.integers(20_000, 60_000)), k=case)
    else:
        pr = dg.make_gauss2d_x2(int(rng.integers(96, 160)), k=case)
    kw0 = dict(grid=pr.grid) if pr.grid is not None else dict(y=pr.t)
    ref = jf.curve_fit(pr.model, pr.z, p0=pr.p0, **kw0)
    comms = jf.Comm.create_local(R, 0)
    if pr.grid is not None:
        W, H = pr.grid[0], pr.grid[1]
        bands = [dg.shard_rows(H, R, r) for r in range(R)]
        zs = [torch.as_tensor(pr.z[r0 * W:r1 * W]).cuda() for r0, r1 in bands]
        kws = [dict(grid=(W, r1 - r0, r0)) for r0, r1 in bands]
    else:
        rngs = [dg.shard_range(pr.m, R, r) for r in range(R)]
        zs = [torch.as_tensor(pr.z[a:b]).cuda() for a, b in rngs]
        kws = [dict(y=torch.as_tensor(pr.t[a:b]).cuda()) for a, b in rngs]
    torch.cuda.synchronize()
    try:
        def fn(r, s):
            return jf.curve_fit(pr.model, zs[r], p0=pr.p0, comm=comms[r], m_global=pr.m, stream=s.cuda_stream,
                                **kws[r])
        outs = _run_ranks(R, fn)
    finally:
        for c in comms:
            c.destroy()
    for o in outs:
        assert (o.status, o.nfev, o.njev, o.nit) == (ref.status, ref.nfev, ref.njev, ref.nit), pr.name
        assert np.allclose(o.x, ref.x, rtol=1e-6), pr.name
    for o in outs[1:]:
        assert np.array_equal(o.x, outs[0].x) and o.cost == outs[0].cost

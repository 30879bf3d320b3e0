"""Out-of-bounds guards (the sanitizer substitute: compute-sanitizer is not
available on the GPU pool).  Every input array is placed inside a larger
device buffer filled with NaN, every device output inside a canary-filled
buffer: a kernel that reads one element outside its input sees a NaN (the
non-finite count becomes non-zero and the result changes), one that writes
outside its output overwrites a canary.  Each guarded call must equal the
unguarded call bitwise and leave the canaries intact; offsets cover 16-byte
aligned inputs (bulk-copy path of the moment J-pass) and 8-byte offsets (the
per-lane staging path), ragged tails and several tiles."""
import numpy as np
import pytest

import datagen as dg

jf = pytest.importorskip("paper_2208_12187_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

GUARD = 4096  # doubles of NaN on each side
CANARY = 1.2345678e300


def guarded(a, off):
    """a (host array) copied into the middle of a NaN-filled device buffer at
    element offset GUARD + off; returns (view, whole buffer)."""
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    buf = torch.full((a.size + 2 * GUARD + 8,), float("nan"), dtype=torch.float64, device="cuda")
    buf[GUARD + off:GUARD + off + a.size] = torch.as_tensor(a).cuda()
    return buf[GUARD + off:GUARD + off + a.size], buf


def assert_guard_intact(buf, lo, hi):
    g = buf.cpu().numpy()
    assert np.isnan(g[:lo]).all() and np.isnan(g[hi:]).all()


def _pass_cases():
    return [
        ("gauss2d 300x97", dg.make_gauss2d(300, H=97, seed=3), {}),
        ("gauss2d 1024x40", dg.make_gauss2d(1024, H=40, seed=3), {}),
        ("gauss2d odd W", dg.make_gauss2d(301, H=33, seed=4), {}),
        ("gauss2d_x2 256x64", dg.make_gauss2d_x2(256, H=64, seed=5), {}),
        ("exp_decay 3001", dg.make_exp_decay(m=3001), {}),
        ("gauss1d 70001", dg.make_gauss1d(70001), {}),
        ("linear 517", dg.make_linear(517), {}),
    ]


def _kw(pr):
    return {"grid": pr.grid} if pr.grid is not None else {}


@pytest.mark.parametrize("off", [0, 1])
@pytest.mark.parametrize("case", range(7))
def test_passes_read_only_their_inputs(case, off):
    name, pr, _ = _pass_cases()[case]
    ref = jf.jpass(pr.model, pr.z, pr.p0, **_kw(pr), **({"y": pr.t} if pr.t is not None else {}))
    zg, zbuf = guarded(pr.z, off)
    kw = _kw(pr)
    if pr.t is not None:
        tg, tbuf = guarded(pr.t, off)
        kw["y"] = tg
    got = jf.jpass(pr.model, zg, pr.p0, **kw)
    assert got[3] == 0 and ref[3] == 0, name
    assert got[0] == ref[0] and np.array_equal(got[1], ref[1]) and np.array_equal(got[2], ref[2]), name
    c_r, bad_r = jf.residual_pass(pr.model, zg, pr.p0, **kw)
    assert bad_r == 0 and c_r == jf.residual_pass(pr.model, pr.z, pr.p0, **_kw(pr),
                                                  **({"y": pr.t} if pr.t is not None else {}))[0]
    assert_guard_intact(zbuf, GUARD + off, GUARD + off + pr.m)


def test_weighted_pass_reads_only_its_inputs():
    pr = dg.make_gauss2d(300, H=50, seed=3)
    sig = 0.1 + 0.01 * np.arange(pr.m) / pr.m
    ref = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid, sigma=sig)
    zg, _ = guarded(pr.z, 1)
    sg, _ = guarded(sig, 3)
    got = jf.jpass(pr.model, zg, pr.p0, grid=pr.grid, sigma=sg)
    assert got[3] == 0 and got[0] == ref[0] and np.array_equal(got[2], ref[2])


def test_pass_device_writes_only_its_output():
    pr = dg.make_gauss2d(300, H=97, seed=3)
    zd = torch.as_tensor(pr.z).cuda()
    xd = torch.as_tensor(pr.p0).cuda()
    out = torch.full((37 + 2 * 64,), CANARY, dtype=torch.float64, device="cuda")
    jf.pass_device(pr.model, zd, xd, out[64:64 + 37], grid=pr.grid)
    jf.pass_device(pr.model, zd, xd, out[64:64 + 2], grid=pr.grid, residual_only=True)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert np.all(o[:64] == CANARY) and np.all(o[64 + 37:] == CANARY)


@pytest.mark.parametrize("solver", ["auto", "tsqr"])
@pytest.mark.parametrize("use_graph", [True, False])
def test_fits_read_only_their_inputs(solver, use_graph):
    pr = dg.make_gauss2d(256, seed=3)
    ref = jf.curve_fit(pr.model, torch.as_tensor(pr.z).cuda(), p0=pr.p0, grid=pr.grid, solver=solver,
                       use_graph=use_graph)
    zg, zbuf = guarded(pr.z, 1)
    res = jf.curve_fit(pr.model, zg, p0=pr.p0, grid=pr.grid, solver=solver, use_graph=use_graph)
    assert (res.status, res.nfev, res.njev) == (ref.status, ref.nfev, ref.njev)
    assert np.array_equal(res.x, ref.x) and res.cost == ref.cost
    assert_guard_intact(zbuf, GUARD + 1, GUARD + 1 + pr.m)
    p1 = dg.make_gauss1d(20000)  # dual-number kernels + solver kernel, explicit t
    ref = jf.curve_fit(p1.model, p1.z, y=p1.t, p0=p1.p0, solver=solver, use_graph=use_graph)
    zg, _ = guarded(p1.z, 3)
    tg, _ = guarded(p1.t, 5)
    res = jf.curve_fit(p1.model, zg, y=tg, p0=p1.p0, solver=solver, use_graph=use_graph)
    assert np.array_equal(res.x, ref.x) and res.nfev == ref.nfev


def test_small_and_batched_fits_read_only_their_inputs():
    p1 = dg.make_exp_decay(m=1000)
    ref = jf.curve_fit(p1.model, p1.z, y=p1.t, p0=p1.p0)
    zg, _ = guarded(p1.z, 1)
    tg, _ = guarded(p1.t, 2)
    res = jf.curve_fit(p1.model, zg, y=tg, p0=p1.p0)
    assert np.array_equal(res.x, ref.x) and res.nfev == ref.nfev
    pb = [dg.make_exp_decay(m=200, k=k) for k in range(37)]
    zb = np.stack([p.z for p in pb])
    rb_ref = jf.curve_fit_batch("exp_decay", zb, y=pb[0].t, shared_y=True, p0=np.ones((37, 3)))
    zg, zbuf = guarded(zb, 1)
    tg, _ = guarded(pb[0].t, 1)
    rb = jf.curve_fit_batch("exp_decay", zg.reshape(37, 200), y=tg, shared_y=True, p0=np.ones((37, 3)))
    assert np.array_equal(rb.x, rb_ref.x) and np.array_equal(rb.nfev, rb_ref.nfev)
    assert np.all(rb.status > 0)
    assert_guard_intact(zbuf, GUARD + 1, GUARD + 1 + zb.size)

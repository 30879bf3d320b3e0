"""GPU parity of the data-parallel passes against the
oracle (oracle/passes.py), called through the C ABI.

Tolerances (north star: per-pass cost, gradient and Gram to 1e-10 relative,
fp64), Cauchy-Schwarz-normalised so near-zero entries are well posed
(SURVEY §8(c) c.3): |dcost| <= 1e-10 cost, |dg_j| <= 1e-10 sqrt(G_jj 2 cost),
|dG_jk| <= 1e-10 sqrt(G_jj G_kk)."""
import math

import numpy as np
import pytest

import datagen as dg
from oracle import passes as orp

jf = pytest.importorskip("paper_2208_12187_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = 1e-10


def check_pass(gpu, ref, tol=TOL):
    c, g, G, bad = gpu
    cr, gr, Gr, badr = ref
    assert bad == badr
    assert abs(c - cr) <= tol * cr
    d = np.sqrt(np.diag(Gr))
    assert np.all(np.abs(g - gr) <= tol * d * math.sqrt(2 * cr) + 1e-300)
    assert np.all(np.abs(G - Gr) <= tol * np.outer(d, d) + 1e-300)
    assert np.array_equal(G, G.T)


def _x_near(pr, k):
    if k == 0:
        return pr.p0
    if k == 1:
        return pr.truth
    rng = np.random.default_rng(k)
    x = pr.truth * (1 + rng.uniform(-0.3, 0.3, pr.n))
    return x


CASES = [
    ("exp_decay m=1000", lambda: dg.make_exp_decay()),
    ("exp_decay ragged", lambda: dg.make_exp_decay(m=296 * 256 * 3 + 77)),
    ("gauss1d m=1000", lambda: dg.make_gauss1d(1000)),
    ("gauss1d ragged", lambda: dg.make_gauss1d(256 * 1000 + 13)),
    ("linear", lambda: dg.make_linear(m=5001)),
    ("gauss2d W=64", lambda: dg.make_gauss2d(64)),
    ("gauss2d W=1000x777", lambda: dg.make_gauss2d(1000, H=777)),
    ("gauss2d W=1024", lambda: dg.make_gauss2d(1024)),
    # the moment kernel's whole-task fast path (rows of 4 x 512-pixel chunks),
    # and rows mixing whole tasks with a shorter row-end task
    ("gauss2d W=2048x48", lambda: dg.make_gauss2d(2048, H=48)),
    ("gauss2d W=2600x37", lambda: dg.make_gauss2d(2600, H=37)),
    ("gauss2d_x2 W=96", lambda: dg.make_gauss2d_x2(96)),
    ("gauss2d_x2 W=700x333", lambda: dg.make_gauss2d_x2(700, H=333)),
    ("gauss2d_x2 W=2048x40", lambda: dg.make_gauss2d_x2(2048, H=40)),
    ("gauss2d_x2 W=2600x31", lambda: dg.make_gauss2d_x2(2600, H=31)),
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("xk", [0, 1, 2])
def test_jpass_matches_oracle_implicit_coords(name, make, xk):
    pr = make()
    x = _x_near(pr, xk)
    ref = orp.jpass(pr.model, pr.coords(), pr.z, x)
    if pr.grid is not None:
        gpu = jf.jpass(pr.model, pr.z, x, grid=pr.grid)
    elif "t0" in pr.meta:
        gpu = jf.jpass(pr.model, pr.z, x, t0=pr.meta["t0"], dt=pr.meta["dt"])
    else:
        gpu = jf.jpass(pr.model, pr.z, x, y=pr.t)
    check_pass(gpu, ref)


@pytest.mark.parametrize("name,make", CASES[::2], ids=[c[0] for c in CASES[::2]])
def test_jpass_matches_oracle_explicit_coords_device_inputs(name, make):
    pr = make()
    x = _x_near(pr, 2)
    y = pr.coords()
    ref = orp.jpass(pr.model, y, pr.z, x)
    yd = torch.as_tensor(np.concatenate(y) if isinstance(y, tuple) else y).cuda()
    gpu = jf.jpass(pr.model, torch.as_tensor(pr.z).cuda(), x, y=yd)
    check_pass(gpu, ref)


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_residual_pass_matches_oracle(name, make):
    pr = make()
    x = _x_near(pr, 2)
    cr, badr = orp.residual_pass(pr.model, pr.coords(), pr.z, x)
    kw = dict(grid=pr.grid) if pr.grid is not None else dict(y=pr.t)
    c, bad = jf.residual_pass(pr.model, pr.z, x, **kw)
    assert bad == badr and abs(c - cr) <= TOL * cr


def test_nonfinite_counts_and_weighted_pass():
    pr = dg.make_gauss1d(50_000)
    z = pr.z.copy()
    z[[5, 40_000, 49_999]] = np.nan
    _, _, _, bad = jf.jpass(pr.model, z, pr.p0, y=pr.t)
    c, bad2 = jf.residual_pass(pr.model, z, pr.p0, y=pr.t)
    assert bad == 3 and bad2 == 3 and not np.isfinite(c)
    sig = np.random.default_rng(1).uniform(0.5, 2.0, pr.m)
    ref = orp.jpass(pr.model, pr.t, pr.z, pr.p0, sigma=sig)
    check_pass(jf.jpass(pr.model, pr.z, pr.p0, y=pr.t, sigma=sig), ref)


@pytest.mark.parametrize("make", [lambda: dg.make_gauss2d(300, H=77), lambda: dg.make_gauss2d_x2(160, H=90)],
                         ids=["gauss2d", "gauss2d_x2"])
def test_weighted_grid_pass_uses_dual_kernel_shape(make):
    """Weighted implicit-grid passes run the dual-number kernels (the moment
    kernels are unweighted) with their own launch shape."""
    pr = make()
    sig = np.random.default_rng(3).uniform(0.5, 2.0, pr.m)
    ref = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0, sigma=sig)
    check_pass(jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid, sigma=sig), ref)


@pytest.mark.parametrize("make", [lambda: dg.make_gauss2d(64, H=17000), lambda: dg.make_gauss2d_x2(64, H=15000)],
                         ids=["gauss2d", "gauss2d_x2"])
def test_moment_kernel_task_rounds(make):
    """Tall images give a block more tasks than its slots: the moment kernels
    run them in rounds (fixed order) — same result, bitwise reproducible."""
    pr = make()
    ref = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
    a = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    check_pass(a, ref)
    b = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_nonfinite_counts_moment_kernel():
    """Non-finite residuals in whole-task (fast path) and row-end chunks are
    counted exactly (per-chunk sum r^2 test + replay) in the moment J-pass."""
    pr = dg.make_gauss2d(2600, H=23)
    z = pr.z.copy()
    idx = [0, 17, 2047, 2048, 2599, 2600 * 5 + 1000, 2600 * 22 + 2599]
    z[idx[:4]] = np.nan
    z[idx[4:]] = np.inf
    _, _, _, bad = jf.jpass(pr.model, z, pr.p0, grid=pr.grid)
    _, bad_r = jf.residual_pass(pr.model, z, pr.p0, grid=pr.grid)
    assert bad == len(idx) and bad_r == len(idx)
    pr2 = dg.make_gauss2d_x2(2600, H=23)  # the two-component moment kernel
    z2 = pr2.z.copy()
    z2[idx[:4]] = np.nan
    z2[idx[4:]] = np.inf
    assert jf.jpass(pr2.model, z2, pr2.p0, grid=pr2.grid)[3] == len(idx)


def test_pass_is_bitwise_deterministic():
    pr = dg.make_gauss2d(512)
    a = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    b = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_pass_device_async_matches_sync():
    """pass_device (device x) against jpass (host x).  With opts.x_host the
    moment J-pass takes the same host-computed prologue as jpass: bitwise
    equal; without it the kernel computes the prologue itself (device cos /
    sin / exp, which may differ from the host's in the last bit): parity."""
    pr = dg.make_gauss2d(300)
    zd = torch.as_tensor(pr.z).cuda()
    xd = torch.as_tensor(pr.p0).cuda()
    kv = torch.zeros(37, dtype=torch.float64, device="cuda")
    kv2 = torch.zeros(37, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    jf.pass_device(pr.model, zd, xd, kv, grid=pr.grid, stream=s.cuda_stream, x_host=pr.p0)
    jf.pass_device(pr.model, zd, xd, kv2, grid=pr.grid, stream=s.cuda_stream)
    torch.cuda.synchronize()
    c, g, G, bad = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    k = kv.cpu().numpy()
    assert k[-2] * 0.5 == c and k[-1] == bad
    k2 = kv2.cpu().numpy()
    assert abs(k2[-2] * 0.5 - c) <= TOL * c and k2[-1] == bad
    ref = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
    check_pass((0.5 * k2[-2], g, G, int(k2[-1])), ref)


@pytest.mark.slow
@pytest.mark.parametrize("xk", [0, 1])
def test_full_size_T_pass_matches_oracle(xk):
    """BASELINE target T (4096^2, seed 6) at the bench's launch configuration."""
    pr = dg.make_gauss2d(4096, seed=6)
    x = pr.p0 if xk == 0 else pr.truth
    ref = orp.jpass(pr.model, pr.coords(), pr.z, x)
    check_pass(jf.jpass(pr.model, torch.as_tensor(pr.z).cuda(), x, grid=pr.grid), ref)
    cr, _ = orp.residual_pass(pr.model, pr.coords(), pr.z, x)
    c, _ = jf.residual_pass(pr.model, pr.z, x, grid=pr.grid)
    assert abs(c - cr) <= TOL * cr


@pytest.mark.slow
def test_full_size_C5_pass_matches_oracle_on_row_band():
    """C5 (8192^2, n=13): the pass over a row band, as one rank of 8 sees it."""
    W = 8192
    pr = dg.make_gauss2d_x2(W, seed=5)
    r0, r1 = dg.shard_rows(W, 8, 3)
    z = pr.z[r0 * W:r1 * W]
    X, Y = dg.grid_coords(W, r1 - r0, r0)
    ref = orp.jpass(pr.model, (X, Y), z, pr.p0)
    check_pass(jf.jpass(pr.model, torch.as_tensor(z).cuda(), pr.p0, grid=(W, r1 - r0, r0)), ref)


def _alt_coefs(sx, sy, th):
    """(a, 2b, c2) of the rotated Gaussian's quadratic form."""
    C, S = math.cos(th), math.sin(th)
    return (C * C / (2 * sx * sx) + S * S / (2 * sy * sy),
            2 * S * C * (1 / (2 * sy * sy) - 1 / (2 * sx * sx)),
            S * S / (2 * sx * sx) + C * C / (2 * sy * sy))


@pytest.mark.parametrize("name,make", [c for c in CASES if c[0].startswith("gauss2d")],
                         ids=[c[0] for c in CASES if c[0].startswith("gauss2d")])
def test_jpass_first_stage_alt_coordinates(name, make):
    """Stage one of the two-stage chain rule (jf_models.cuh PreGauss2D) alone:
    with the map T^T M T switched off (JF_FLAG_ALT_COORDS), the pass returns
    the Gram of [J_alt | r] whose shape columns are d h / d(a, 2b, c2) =
    -A E (dx^2, dx dy, dy^2) — written out here from the quadratic form, so a
    wrong stage-two map cannot hide behind a compensating stage-one error."""
    pr = make()
    X, Y = pr.coords()
    x = pr.p0
    cols = []
    for B in range(0, pr.n - 1, 6):
        A, x0, y0 = x[B:B + 3]
        a, b2, c2 = _alt_coefs(*x[B + 3:B + 6])
        dx, dy = X - x0, Y - y0
        E = np.exp(-(a * dx * dx + b2 * dx * dy + c2 * dy * dy))
        AE = A * E
        cols += [E, AE * (2 * a * dx + b2 * dy), AE * (b2 * dx + 2 * c2 * dy), -AE * dx * dx, -AE * dx * dy, -AE * dy * dy]
    Ja = np.stack(cols + [np.ones_like(X)], 1)
    r = dg.render(pr.model, (X, Y), x) - pr.z
    ref = (0.5 * float(r @ r), Ja.T @ r, Ja.T @ Ja, 0)
    check_pass(jf.jpass(pr.model, pr.z, x, grid=pr.grid, alt_coords=True), ref, tol=1e-9)


EDGE = [  # (A, x0, y0, sx, sy, theta, off) on a 4096-wide image
    ("narrow 2px", (1.5, 2047.3, 511.7, 2.0, 2.5, 0.4, 0.2)),
    ("needle 3x1500px", (1.2, 1900.0, 500.0, 3.0, 1500.0, 0.3, 0.1)),
    ("off-image centre", (2.0, -300.0, 1300.0, 400.0, 250.0, 2.1, 0.3)),
    ("edge centre", (1.0, 4095.0, 0.0, 60.0, 900.0, 1.2, 0.05)),
    ("wide flat", (0.8, 2000.0, 600.0, 30000.0, 20000.0, 0.7, 0.4)),
    ("aspect 10 at the moment form's limit", (1.3, 2100.0, 480.0, 60.0, 600.0, 0.9, 0.25)),
    ("width 50 at the moment form's limit", (1.1, 1500.0, 700.0, 50.0, 70.0, 2.5, 0.15)),
]


@pytest.mark.slow
@pytest.mark.parametrize("name,truth", EDGE, ids=[e[0] for e in EDGE])
def test_jpass_edge_shapes_full_width(name, truth):
    """The moment kernel's recurrence / direct-evaluation switch (exponent
    guards q < 600, |argR| < 300 per row segment) at T's row length: narrow,
    needle-like, off-image and edge-centred peaks and a nearly flat one, on a
    4096 x 1024 band, at the truth and a perturbed point."""
    pr = dg.make_gauss2d_at(4096, 1024, truth)
    for x in (pr.truth, pr.truth * np.array([1.05, 1.0, 1.0, 1.3, 0.8, 1.0, 1.1]) + np.array([0, 2.5, -1.5, 0, 0, 0.05, 0])):
        ref = orp.jpass(pr.model, pr.coords(), pr.z, x)
        check_pass(jf.jpass(pr.model, torch.as_tensor(pr.z).cuda(), x, grid=pr.grid), ref)
        cr, _ = orp.residual_pass(pr.model, pr.coords(), pr.z, x)
        c, _ = jf.residual_pass(pr.model, pr.z, x, grid=pr.grid)
        assert abs(c - cr) <= TOL * cr


@pytest.mark.parametrize("name,truth", EDGE, ids=[e[0] for e in EDGE])
def test_jpass_edge_shapes_small(name, truth):
    """The same shapes scaled to a 640 x 77 image (ragged row ends)."""
    s = 640 / 4096
    t = np.array(truth) * np.array([1, s, s, s, s, 1, 1])
    t[3:5] = np.maximum(t[3:5], [0.7, 0.9])  # (sx == sy would make the theta column identically 0)
    pr = dg.make_gauss2d_at(640, 77, t)
    ref = orp.jpass(pr.model, pr.coords(), pr.z, pr.truth)
    check_pass(jf.jpass(pr.model, pr.z, pr.truth, grid=pr.grid), ref)


@pytest.mark.parametrize("comp2", [(1.0, 300.0, 40.0, 2.5, 2.0, 0.3), (0.9, 420.0, 30.0, 5.0, 120.0, 1.0),
                                   (1.2, 380.0, 35.0, 60.0, 90.0, 2.0)],
                         ids=["narrow", "needle", "moderate"])
def test_jpass_two_gaussians_edge_shapes(comp2):
    """The n = 13 moment kernel's accuracy switch: a narrow or elongated second
    component sends the pass to the dual-number body; a moderate one stays."""
    W, H = 600, 70
    X, Y = dg.grid_coords(W, H)
    p1 = np.array([1.5, 150.0, 30.0, 80.0, 100.0, 0.7])
    truth = np.concatenate([p1, comp2, [0.2]])
    z = dg.render("gauss2d_rot_x2", (X, Y), truth) + 0.1 * np.random.default_rng(8).standard_normal(W * H)
    ref = orp.jpass("gauss2d_rot_x2", (X, Y), z, truth)
    check_pass(jf.jpass("gauss2d_rot_x2", z, truth, grid=(W, H, 0)), ref)


@pytest.mark.parametrize("W", [1, 2, 31, 33, 511, 512, 513, 1000, 2049])
@pytest.mark.parametrize("H", [1, 3, 17])
def test_moment_pass_odd_shapes(W, H):
    """The n = 7 moment J-pass (bulk-copy ring, chunk-granular warp split) on
    shapes around its chunk (512 px) and lane (32 px) granularity: fewer
    chunks than warps, one-row images, partial row-end chunks, widths below
    one lane group.  A wide peak keeps the moment form (not the dual-number
    fallback); pixel centres off the peak test the exp-per-point row ends."""
    truth = np.array([1.3, 0.37 * W, 0.61 * H, 80.0, 55.0, 0.4, 0.25])
    pr = dg.make_gauss2d_at(W, H, truth)
    ref = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
    check_pass(jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid), ref)
    zd = torch.as_tensor(pr.z).cuda()  # device input (16-byte aligned: bulk copies when W is even)
    check_pass(jf.jpass(pr.model, zd, pr.p0, grid=pr.grid), ref)


@pytest.mark.parametrize("W,H", [(1, 1), (2, 3), (33, 17), (257, 1), (1000, 3)])
def test_moment2_pass_odd_shapes(W, H):
    """The n = 13 moment J-pass on images narrower than a task / a chunk."""
    truth = np.array([1.3, 0.37 * W, 0.61 * H, 80.0, 55.0, 0.4, 0.9, 0.55 * W, 0.3 * H, 60.0, 90.0, 1.1, 0.25])
    X, Y = dg.grid_coords(W, H)
    z = dg.render("gauss2d_rot_x2", (X, Y), truth) + 0.1 * np.random.default_rng(3).standard_normal(W * H)
    ref = orp.jpass("gauss2d_rot_x2", (X, Y), z, truth)
    check_pass(jf.jpass("gauss2d_rot_x2", z, truth, grid=(W, H, 0)), ref)


@pytest.mark.slow
def test_full_size_C2_pass_matches_oracle():
    """BASELINE config 2 at the top of its length sweep (1D Gaussian, m = 1e7,
    explicit t): the dual-number J-pass and the r-pass at p0 against the oracle."""
    pr = dg.make_gauss1d(10_000_000)
    ref = orp.jpass(pr.model, pr.t, pr.z, pr.p0)
    check_pass(jf.jpass(pr.model, pr.z, pr.p0, y=pr.t), ref)
    cr, _ = orp.residual_pass(pr.model, pr.t, pr.z, pr.p0)
    c, _ = jf.residual_pass(pr.model, pr.z, pr.p0, y=pr.t)
    assert abs(c - cr) <= TOL * cr


@pytest.mark.slow
@pytest.mark.parametrize("W,H", [(2600, 7200), (8192, 8192)])
def test_moment2_sub_runs_equal_dual_number_pass(W, H):
    """Blocks with more tasks than the n = 13 moment kernel's slots run them
    as sub-runs (W = 2600, H = 7200: two; the full C5 image: more) — sizes the
    oracle cannot reduce in test time.  The property that holds at any size:
    the moment form equals the dual-number rank-1 pass (the weighted kernel
    with sigma = 1, pinned to the oracle in the weighted-pass tests) to the
    parity tolerance, on the same device data."""
    pr = dg.make_gauss2d_x2(W, seed=5, H=H)
    zd = torch.as_tensor(pr.z).cuda()
    ones = torch.ones(pr.m, dtype=torch.float64, device="cuda")
    a = jf.jpass(pr.model, zd, pr.p0, grid=pr.grid)
    b = jf.jpass(pr.model, zd, pr.p0, grid=pr.grid, sigma=ones)
    check_pass(a, b)

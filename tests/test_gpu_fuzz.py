"""Seeded random passes against the oracle (1e-10 per pass, the north-star
tolerance): random models, shapes (including ragged tails, one-row and
one-column images, fewer points than lanes), parameter points (wide, narrow,
elongated, rotated, off-centre and off-image peaks — both the moment form and
its dual-number fallback), weights, host or device inputs, residual passes.
Generated from a fixed seed: the same cases every run."""
import math

import numpy as np
import pytest

import datagen as dg
from oracle import passes as orp
from oracle import trf as otrf

jf = pytest.importorskip("paper_2208_12187_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = 1e-10
N_CASES = 240


def _case(k):
    rng = np.random.default_rng([2208, 12187, k])
    model = ["exp_decay", "gauss1d", "linear", "gauss2d_rot", "gauss2d_rot", "gauss2d_rot", "gauss2d_rot_x2"][k % 7]
    if model in ("gauss2d_rot", "gauss2d_rot_x2"):
        W = int(rng.choice([1, 7, 32, 33, 100, 511, 512, 700, 1500]))
        H = int(rng.choice([1, 2, 5, 40, 129]))
        X, Y = dg.grid_coords(W, H)

        def comp():
            A = rng.uniform(0.2, 3.0)
            x0 = rng.uniform(-0.3, 1.3) * W
            y0 = rng.uniform(-0.3, 1.3) * H
            sx = np.exp(rng.uniform(np.log(2.0), np.log(600.0)))
            sy = np.exp(rng.uniform(np.log(2.0), np.log(600.0)))
            th = rng.uniform(-np.pi, np.pi)
            return [A, x0, y0, sx, sy, th]
        x = comp() + (comp() if model == "gauss2d_rot_x2" else []) + [rng.uniform(-0.5, 0.5)]
        coords = (X, Y)
        kw = dict(grid=(W, H, 0))
        m = W * H
    else:
        m = int(rng.choice([1, 5, 31, 33, 1000, 4097, 60001]))
        t = np.sort(rng.uniform(0.0, 3.0, m)) if rng.uniform() < 0.5 else np.linspace(0.0, 3.0, m)
        x = {"exp_decay": [rng.uniform(0.5, 3), rng.uniform(0.1, 2), rng.uniform(-1, 1)],
             "gauss1d": [rng.uniform(0.5, 2), rng.uniform(0.5, 2.5), rng.uniform(0.05, 1.0), rng.uniform(-1, 1)],
             "linear": [rng.uniform(-2, 2), rng.uniform(-2, 2)]}[model]
        coords = t
        kw = dict(y=t)
    x = np.array(x)
    z = dg.render(model, coords, x * (1 + 0.05 * rng.standard_normal(x.size))) + 0.1 * rng.standard_normal(m)
    sigma = rng.uniform(0.05, 0.3, m) if rng.uniform() < 0.25 else None
    on_device = rng.uniform() < 0.5
    return model, coords, z, x, kw, sigma, on_device


def _check(gpu, ref, what):
    c, g, G, bad = gpu
    cr, gr, Gr, badr = ref
    assert bad == badr, what
    assert abs(c - cr) <= TOL * cr, what
    # (a column whose entries are all far below the largest column's — a peak
    # entirely off the image, exp(-q) ~ 1e-170 — has a Gram diagonal that
    # underflows to 0 while J^T r does not: Cauchy-Schwarz normalisation with
    # a floor 1e-150 of the largest column norm, numerically zero)
    d = np.sqrt(np.diag(Gr))
    d = np.maximum(d, 1e-150 * np.max(d))
    assert np.all(np.abs(g - gr) <= TOL * d * math.sqrt(2 * cr) + 1e-300), what
    assert np.all(np.abs(G - Gr) <= TOL * np.outer(d, d) + 1e-300), what


@pytest.mark.parametrize("k", range(N_CASES))
def test_random_pass_matches_oracle(k):
    model, coords, z, x, kw, sigma, on_device = _case(k)
    what = f"case {k}: {model} m={z.size} {kw.get('grid', '')} sigma={sigma is not None} device={on_device}"
    ref = orp.jpass(model, coords, z, x, sigma=sigma)
    cr, badr = orp.residual_pass(model, coords, z, x, sigma=sigma)
    if on_device:
        z = torch.as_tensor(z).cuda()
        if "y" in kw:
            kw = dict(y=torch.as_tensor(kw["y"]).cuda())
        if sigma is not None:
            sigma = torch.as_tensor(sigma).cuda()
    _check(jf.jpass(model, z, x, sigma=sigma, **kw), ref, what)
    c, bad = jf.residual_pass(model, z, x, sigma=sigma, **kw)
    assert bad == badr and abs(c - cr) <= TOL * cr, what


def _fit_case(k):
    rng = np.random.default_rng([2208, 7, k])
    kind = k % 5
    if kind == 0:
        return dg.make_exp_decay(m=int(rng.integers(50, 3000)), k=k)
    if kind == 1:
        return dg.make_gauss1d(int(rng.integers(500, 200_000)), k=k)
    if kind == 2:
        return dg.make_gauss2d(int(rng.integers(48, 320)), k=k, H=int(rng.integers(48, 320)))
    if kind == 3:
        return dg.make_gauss2d_bounded(int(rng.integers(64, 256)), "abc"[k % 3], k=k)
    return dg.make_gauss2d_x2(int(rng.integers(64, 200)), k=k)


@pytest.mark.parametrize("k", range(30))
def test_random_fit_matches_oracle(k):
    """Seeded fits drawn from the BASELINE recipes (datagen, other draws and
    sizes): the CUDA fit (graph driver, solver AUTO) against the oracle's TRF —
    same status and counts, x to 1e-6."""
    pr = _fit_case(k)
    ref = otrf.fit(pr.model, pr.coords(), pr.z, pr.p0, pr.lb, pr.ub)
    kw = dict(grid=pr.grid) if pr.grid is not None else dict(y=pr.t)
    res = jf.curve_fit(pr.model, pr.z, p0=pr.p0, lb=pr.lb, ub=pr.ub, **kw)
    what = f"case {k}: {pr.name}"
    assert (res.status, res.nfev, res.njev, res.nit) == (ref["status"], ref["nfev"], ref["njev"], ref["nit"]), what
    x = ref["x"]
    assert np.all(np.abs(res.x - x) <= 1e-6 * np.maximum(np.abs(x), 1e-3 * np.max(np.abs(x)))), what


@pytest.mark.parametrize("mode", ["tsqr", "conservative", "hostloop", "capacity", "weighted"])
@pytest.mark.parametrize("k", range(8))
def test_random_fit_modes_match_oracle(k, mode):
    """The same seeded fits through the other fit paths: TSQR solver,
    conservative policy (r-pass per trial), host-driven loop, a capacity-sized
    graph (App. A masking without dummy data) and per-point weights."""
    pr = _fit_case(100 + k)
    kw = dict(grid=pr.grid) if pr.grid is not None else dict(y=pr.t)
    sigma = None
    if mode == "weighted":
        sigma = np.random.default_rng([7, k]).uniform(0.05, 0.2, pr.m)
        kw["sigma"] = sigma
    elif mode == "tsqr":
        kw["solver"] = "tsqr"
    elif mode == "conservative":
        kw["policy"] = "conservative"
    elif mode == "hostloop":
        kw["use_graph"] = False
    elif mode == "capacity":
        kw["capacity"] = pr.m + 12345
    ref = otrf.fit(pr.model, pr.coords(), pr.z, pr.p0, pr.lb, pr.ub, sigma=sigma)
    res = jf.curve_fit(pr.model, pr.z, p0=pr.p0, lb=pr.lb, ub=pr.ub, **kw)
    what = f"case {k} {mode}: {pr.name}"
    assert (res.status, res.nfev, res.njev, res.nit) == (ref["status"], ref["nfev"], ref["njev"], ref["nit"]), what
    x = ref["x"]
    assert np.all(np.abs(res.x - x) <= 1e-6 * np.maximum(np.abs(x), 1e-3 * np.max(np.abs(x)))), what

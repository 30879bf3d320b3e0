"""Pins for oracle/trf.py (Alg. 1-3, Eq. 9-15, App. B, readings R3-R27).

Pinned against: closed forms (linear least squares; the J=I subproblem),
the Moré-Sorensen conditions (Eq. 9-11), bisection on phi (Eq. 13),
finite differences of phi (R11), Alg. 3's branch table, exact recovery of
noise-free data, and the external library the paper names as its algorithm
(SciPy's TRF, P:42 / P:246): identical nfev/njev/status and x to 1e-10."""
import math

import numpy as np
import pytest
from scipy.optimize import least_squares
from scipy.optimize._lsq import common as sp_common
from scipy.optimize._lsq import trf as sp_trf

import datagen as dg
from oracle import models, trf


def _svd(J):
    U, s, VT = np.linalg.svd(J, full_matrices=False)
    return U, s, VT.T


# --------------------------------------------------------------- subproblem

def test_solve_tr_identity_closed_forms():
    # J = I, r = [3, 4]: p(alpha) = -r / (1 + alpha); ||p|| = Delta at alpha = 5/Delta - 1
    J = np.eye(2)
    r = np.array([3.0, 4.0])
    U, s, V = _svd(J)
    uf = U.T @ r
    p, alpha, it = trf.solve_tr(2, 2, uf, s, V, 1.0, 0.0)
    assert np.allclose(p, [-0.6, -0.8], rtol=0, atol=1e-15)
    assert alpha == pytest.approx(4.0, rel=1e-12) and it == 2
    p, alpha, it = trf.solve_tr(2, 2, uf, s, V, 5.0, 0.0)     # phi(0) = 0: GN step
    assert it == 0 and alpha == 0.0 and np.allclose(p, [-3, -4], atol=1e-15)
    # S:193-199 examples: alpha = 0 -> p = -[1,2]; alpha = 1 -> -[0.5, 1]
    r = np.array([1.0, 2.0])
    U, s, V = _svd(J)
    for a, want in [(0.0, [-1.0, -2.0]), (1.0, [-0.5, -1.0])]:
        suf = s * (U.T @ r)
        assert np.allclose(-V @ (suf / (s * s + a)), want, atol=1e-15)


def test_solve_tr_more_sorensen_and_bisection():
    rng = np.random.default_rng(7)
    for _ in range(200):
        m = int(rng.integers(3, 60))
        n = int(rng.integers(1, min(m, 10) + 1))
        J = rng.standard_normal((m, n)) * rng.uniform(0.1, 10, n)
        r = rng.standard_normal(m)
        U, s, V = _svd(J)
        uf = U.T @ r
        g = J.T @ r
        pgn = np.linalg.lstsq(J, -r, rcond=None)[0]
        Delta = float(np.linalg.norm(pgn)) * rng.uniform(0.05, 0.9)
        p, alpha, it = trf.solve_tr(n, m, uf, s, V, Delta, 0.0)
        assert it > 0 and alpha > 0
        # Eq. 9 residual before the R12 normalisation: solve with the returned alpha
        p_raw = np.linalg.solve(J.T @ J + alpha * np.eye(n), -g)
        assert np.linalg.norm((J.T @ J + alpha * np.eye(n)) @ p_raw + g) <= 1e-8 * np.linalg.norm(g)
        # Eq. 10 (complementarity to sigma = 0.01) and the final normalisation R12
        assert abs(np.linalg.norm(p) - Delta) <= 1e-12 * Delta
        assert abs(np.linalg.norm(p_raw) - Delta) < 0.01 * Delta * 1.0001 + 1e-12
        # bisection root of phi (Eq. 13) lies near alpha (sigma = 0.01 bound, not 1e-6: R9)
        lo, hi = 0.0, float(np.linalg.norm(g)) / Delta
        suf = s * uf
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if trf.phi_and_derivative(mid, suf, s, Delta)[0] > 0:
                lo = mid
            else:
                hi = mid
        assert abs(trf.phi_and_derivative(alpha, suf, s, Delta)[0]) < 0.011 * Delta
        assert alpha == pytest.approx(0.5 * (lo + hi), rel=0.05)


def test_phi_derivative_matches_finite_difference():
    rng = np.random.default_rng(9)
    s = np.sort(rng.uniform(0.1, 5, 6))[::-1]
    suf = rng.standard_normal(6)
    for a in [0.01, 0.3, 2.0, 17.0]:
        h = 1e-6 * a
        fd = (trf.phi_and_derivative(a + h, suf, s, 1.0)[0] - trf.phi_and_derivative(a - h, suf, s, 1.0)[0]) / (2 * h)
        assert trf.phi_and_derivative(a, suf, s, 1.0)[1] == pytest.approx(fd, rel=1e-7)


def test_solve_tr_matches_library_routine():
    """SciPy's solve_lsq_trust_region (the routine P:42 names) on random and
    rank-deficient instances, including warm starts.  Identical iteration
    counts; alpha and p to 1e-12 (the oracle groups Eq. 14 as the paper prints
    it, ((phi+Delta)/Delta)(phi/phi'), SciPy as (phi+Delta)*ratio/Delta)."""
    rng = np.random.default_rng(11)
    for k in range(300):
        m = int(rng.integers(1, 40))
        n = int(rng.integers(1, 9))
        J = rng.standard_normal((m, n))
        if k % 5 == 0 and n > 1:
            J[:, -1] = J[:, 0]                    # rank deficient
        r = rng.standard_normal(m)
        U, s, V = _svd(J)
        uf = U.T @ r
        Delta = 10 ** rng.uniform(-2, 1)
        a0 = 0.0 if k % 3 else float(rng.uniform(0, 3))
        p, a, it = trf.solve_tr(n, m, uf, s, V, Delta, a0)
        p2, a2, it2 = sp_common.solve_lsq_trust_region(n, m, uf, s, V, Delta, initial_alpha=a0)
        assert it == it2
        assert a == pytest.approx(a2, rel=1e-12, abs=0)
        assert np.allclose(p, p2, rtol=1e-12, atol=1e-14 * np.linalg.norm(p2))


def test_solve_tr_survey_goldens():
    # J = diag(1,2), r = [1,1], Delta = 0.1: alpha root 19.068010435056127 (phi within 1% of Delta)
    J = np.diag([1.0, 2.0])
    U, s, V = _svd(J)
    p, a, it = trf.solve_tr(2, 2, U.T @ np.ones(2), s, V, 0.1, 0.0)
    assert a == pytest.approx(19.068010435056127, rel=1e-4)
    assert np.linalg.norm(p) == pytest.approx(0.1, rel=1e-14)
    # rank deficient J = [e1 0] (3x2), r = [1,1,0], Delta = 0.5 -> p = [-0.5, 0]
    J = np.array([[1.0, 0.0], [0.0, 0.0], [0.0, 0.0]])
    U, s, V = _svd(J)
    p, a, it = trf.solve_tr(2, 3, U.T @ np.array([1.0, 1.0, 0.0]), s, V, 0.5, 0.0)
    assert np.allclose(p, [-0.5, 0.0], atol=1e-12)


# ------------------------------------------------------------ Alg. 3 / R14-R16

@pytest.mark.parametrize("args,want", [
    ((1.0, 0.9, 1.0, 0.99, True), (2.0, 0.9)),
    ((1.0, 0.9, 1.0, 0.5, False), (1.0, 0.9)),
    ((1.0, 0.5, 1.0, 0.99, True), (1.0, 0.5)),
    ((1.0, 0.1, 1.0, 2.0, True), (0.5, 0.1)),
    ((1.0, 0.0, 0.0, 0.3, False), (1.0, 1.0)),
    ((1.0, -1.0, 0.0, 0.3, False), (0.075, 0.0)),
])
def test_update_radius_branches(args, want):
    got = trf.update_radius(*args)
    assert got[0] == pytest.approx(want[0], rel=1e-15) and got[1] == pytest.approx(want[1], rel=1e-15)
    assert got == sp_common.update_tr_radius(*args)


def test_termination_rules():
    assert trf.termination(1e-10, 1.0, 1.0, 1.0, 0.5, 1e-8, 1e-8) == 2
    assert trf.termination(1e-10, 1.0, 1.0, 1.0, 0.2, 1e-8, 1e-8) is None   # ratio <= 0.25
    assert trf.termination(1.0, 1.0, 1e-12, 1.0, 0.5, 1e-8, 1e-8) == 3
    assert trf.termination(1e-10, 1.0, 1e-12, 1.0, 0.5, 1e-8, 1e-8) == 4


# ----------------------------------------------------------------- full fits

def test_linear_model_matches_normal_equations():
    """linear least squares has a closed form."""
    pr = dg.make_linear(m=300)
    res = trf.fit(pr.model, pr.t, pr.z, pr.p0)
    A = np.stack([pr.t, np.ones_like(pr.t)], axis=1)
    xs = np.linalg.lstsq(A, pr.z, rcond=None)[0]
    assert np.allclose(res["x"], xs, rtol=1e-10, atol=1e-12)
    assert res["status"] in (1, 2, 3, 4)


@pytest.mark.parametrize("make,canon", [
    (lambda: dg.make_exp_decay(noise=0.0), None),
    (lambda: dg.make_gauss1d(2000, noise=0.0), None),
    (lambda: dg.make_gauss2d(96, noise=0.0), "g2"),
    (lambda: dg.make_gauss2d_x2(96, noise=0.0), "g2x2"),
])
def test_noise_free_exact_recovery(make, canon):
    pr = make()
    p0 = pr.p0 if pr.model != "exp_decay" else pr.truth * np.array([1.2, 0.85, 1.15])
    res = trf.fit(pr.model, pr.coords(), pr.z, p0, xtol=1e-12, ftol=1e-12, gtol=1e-12)
    x = res["x"].copy()
    tr = pr.truth.copy()
    if canon:   # R22: theta modulo pi
        for j in ([5] if canon == "g2" else [5, 11]):
            x[j] = math.remainder(x[j] - tr[j], math.pi) + tr[j]
    assert np.allclose(x, tr, rtol=1e-6, atol=1e-9)


TRAJ_CASES = [
    ("C1", lambda: dg.make_exp_decay()),
    ("C2 m=1000", lambda: dg.make_gauss1d(1000)),
    ("C2 m=20000", lambda: dg.make_gauss1d(20000)),
    ("C3 W=256", lambda: dg.make_gauss2d(256)),
    ("C4a W=256", lambda: dg.make_gauss2d_bounded(256, "a")),
    ("C4b W=256", lambda: dg.make_gauss2d_bounded(256, "b")),
    ("C4c W=256", lambda: dg.make_gauss2d_bounded(256, "c")),
    ("C5 W=128", lambda: dg.make_gauss2d_x2(128)),
    ("linear", lambda: dg.make_linear()),
]


@pytest.mark.parametrize("name,make", TRAJ_CASES, ids=[c[0] for c in TRAJ_CASES])
@pytest.mark.parametrize("x_scale", ["jac", "ones"])
def test_trajectory_matches_scipy_trf(name, make, x_scale):
    pr = make()
    y = pr.coords()
    res = trf.fit(pr.model, y, pr.z, pr.p0, pr.lb, pr.ub, x_scale=x_scale)
    bounds = (-np.inf, np.inf) if pr.lb is None else (pr.lb, pr.ub)
    ref = least_squares(lambda x: models.h(pr.model, y, x) - pr.z, pr.p0,
                        jac=lambda x: models.jac(pr.model, y, x), method="trf",
                        tr_solver="exact", x_scale=(x_scale if x_scale == "jac" else 1.0), bounds=bounds)
    assert (res["status"], res["nfev"], res["njev"]) == (ref.status, ref.nfev, ref.njev)
    assert np.allclose(res["x"], ref.x, rtol=1e-10, atol=1e-12)
    assert res["cost"] == pytest.approx(ref.cost, rel=1e-12)
    if pr.lb is not None:
        assert np.array_equal(res["active_mask"], ref.active_mask)


def test_golden_trajectory_c1_and_c3_values():
    """SURVEY.md §8(c) c.5 goldens (SciPy 1.18.1 outputs on the d.2 recipe)."""
    r = trf.fit("exp_decay", *(lambda p: (p.t, p.z, p.p0))(dg.make_exp_decay()))
    assert (r["status"], r["nfev"], r["njev"]) == (2, 6, 6)
    assert r["cost"] == pytest.approx(19.45078668969252, rel=1e-13)
    assert np.allclose(r["x"], [2.493283850794, 1.306514551524, 0.492743643867], rtol=1e-11)


def test_select_step_gradient_branch_matches_library():
    """The scaled-gradient branch (R20) is reached by no config: crafted case —
    a bound at distance << Delta along p with g nearly normal to the bound.
    Every branch is compared against SciPy's select_step."""
    rng = np.random.default_rng(5)
    seen = set()
    for _ in range(4000):
        n = 3
        m = 8
        Jh = rng.standard_normal((m, n))
        gh = rng.standard_normal(n)
        x = rng.uniform(-1, 1, n)
        lb = x - rng.uniform(1e-3, 1, n)
        ub = x + rng.uniform(1e-3, 1, n)
        d = rng.uniform(0.2, 2, n)
        diag_h = np.abs(rng.standard_normal(n)) * (rng.uniform() < 0.5)
        Delta = 10 ** rng.uniform(-1.5, 0.5)
        p_h = rng.standard_normal(n)
        p_h *= Delta / np.linalg.norm(p_h)
        p = d * p_h
        theta = rng.uniform(0.995, 1.0)
        a = trf.select_step(x, Jh, diag_h, gh, p.copy(), p_h.copy(), d, Delta, lb, ub, theta)
        b = sp_trf.select_step(x, Jh, diag_h, gh, p.copy(), p_h.copy(), d, Delta, lb, ub, theta)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
        seen.add(a[3])
    assert seen == {0, 1, 2, 3}


def test_loose_bounds_equal_unbounded_and_kkt():
    pr = dg.make_gauss2d(128)
    y = pr.coords()
    free = trf.fit(pr.model, y, pr.z, pr.p0)
    lb = np.full(7, -1e9)
    ub = np.full(7, 1e9)
    loose = trf.fit(pr.model, y, pr.z, pr.p0, lb, ub)
    assert np.allclose(loose["x"], free["x"], rtol=1e-6)
    prb = dg.make_gauss2d_bounded(128, "c")
    res = trf.fit(prb.model, prb.coords(), prb.z, prb.p0, prb.lb, prb.ub)
    act = res["active_mask"]
    g = res["grad"]
    assert np.any(act != 0)
    assert np.all(g[act == -1] >= 0) and np.all(g[act == 1] <= 0)


def test_trace_accepted_costs_decrease_and_counts():
    pr = dg.make_gauss2d_bounded(128, "c")
    tr = []
    res = trf.fit(pr.model, pr.coords(), pr.z, pr.p0, pr.lb, pr.ub, trace=tr)
    assert len(tr) == res["nfev"] - 1
    costs = [t[4] for t in tr if t[4] < t[3]]
    assert all(b < a for a, b in zip(costs, costs[1:]))


def test_invalid_inputs():
    pr = dg.make_exp_decay()
    with pytest.raises(trf.FitError) as e:
        trf.fit(pr.model, pr.t, pr.z, pr.p0, lb=[0, 0, 0], ub=[1, 1, 0])
    assert e.value.code == -1
    with pytest.raises(trf.FitError) as e:
        trf.fit(pr.model, pr.t, pr.z, [5.0, 0.5, 0.5], lb=[0, 0, 0], ub=[1, 1, 1])
    assert e.value.code == -2
    z = pr.z.copy()
    z[0] = np.inf
    with pytest.raises(trf.FitError) as e:
        trf.fit(pr.model, pr.t, z, pr.p0)
    assert e.value.code == -3


def test_weighted_fit_equivalences():
    """App. C (Eq. C9/C14-C16): sigma == 1 reproduces the unweighted fit; a
    uniform sigma leaves the minimiser unchanged; sigma == equal to weights
    applied to data by hand gives the same fit."""
    pr = dg.make_gauss1d(3000)
    y = pr.coords()
    a = trf.fit(pr.model, y, pr.z, pr.p0)
    b = trf.fit(pr.model, y, pr.z, pr.p0, sigma=np.ones(pr.m))
    assert np.array_equal(a["x"], b["x"]) and a["nfev"] == b["nfev"]
    c = trf.fit(pr.model, y, pr.z, pr.p0, sigma=np.full(pr.m, 3.0))
    assert np.allclose(c["x"], a["x"], rtol=1e-6)
    sig = np.random.default_rng(3).uniform(0.5, 2.0, pr.m)
    d = trf.fit(pr.model, y, pr.z, pr.p0, sigma=sig)
    ref = least_squares(lambda x: (models.h(pr.model, y, x) - pr.z) / sig, pr.p0,
                        jac=lambda x: models.jac(pr.model, y, x) / sig[:, None], method="trf",
                        tr_solver="exact", x_scale="jac")
    assert d["nfev"] == ref.nfev and np.allclose(d["x"], ref.x, rtol=1e-10)


def test_pcov_matches_curve_fit_library():
    """pcov: the oracle's covariance equals SciPy curve_fit's."""
    from scipy.optimize import curve_fit as sp_curve_fit
    pr = dg.make_gauss1d(2000)
    res = trf.fit(pr.model, pr.t, pr.z, pr.p0)
    f = lambda t, *p: models.h(pr.model, t, np.array(p))
    popt, pc = sp_curve_fit(f, pr.t, pr.z, p0=pr.p0, method="trf", jac=lambda t, *p: models.jac(pr.model, t, np.array(p)),
                            x_scale="jac")
    assert np.allclose(res["x"], popt, rtol=1e-10)
    assert np.allclose(res["pcov"], pc, rtol=1e-8, atol=1e-14 * np.max(np.abs(pc)))
    # full rank: pcov = inv(J^T J) * s^2
    J = models.jac(pr.model, pr.t, res["x"])
    assert np.allclose(res["pcov"], np.linalg.inv(J.T @ J) * 2 * res["cost"] / (pr.m - 4), rtol=1e-9)


def test_default_p0_matches_curve_fit_library():
    """p0 = None (jf.h: 'curve_fit's default initial guess'): the oracle's
    default_p0 equals the point SciPy curve_fit evaluates first — ones
    unbounded; with bounds the midpoint of two finite bounds, lb + 1 / ub - 1
    with one (the point is interior, so least_squares' strict-feasibility
    step leaves it unchanged)."""
    import warnings
    from scipy.optimize import curve_fit as sp_curve_fit
    pr = dg.make_exp_decay()
    cases = [
        (np.full(3, -np.inf), np.full(3, np.inf)),
        (np.array([0.0, -np.inf, -2.0]), np.array([4.0, 3.0, np.inf])),
        (np.array([-1.0, 0.5, -np.inf]), np.array([np.inf, 2.5, 0.0])),
    ]
    for lb, ub in cases:
        first = []

        def f(t, a, b, c):  # curve_fit counts the parameters from the signature
            if not first:
                first.append(np.array([a, b, c]))
            return models.h(pr.model, t, np.array([a, b, c]))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                sp_curve_fit(f, pr.t, pr.z, bounds=(lb, ub), method="trf", max_nfev=1)
            except RuntimeError:
                pass  # max_nfev reached: only the first point matters
        got = trf.default_p0(3, lb, ub)
        assert np.array_equal(got, first[0]), (lb, ub, got, first[0])
        if np.any(np.isfinite(lb)) or np.any(np.isfinite(ub)):
            assert not np.allclose(got, 1.0)  # the bounded rule is exercised


@pytest.mark.parametrize("name,make", [TRAJ_CASES[0], TRAJ_CASES[1], TRAJ_CASES[3]],
                         ids=[TRAJ_CASES[k][0] for k in (0, 1, 3)])
def test_array_x_scale_matches_library(name, make):
    """x_scale given as an array (D = diag(1/x_scale), reading R3): the same
    trajectory as SciPy least_squares(x_scale=array), compared after 3 and
    after all evaluations.  The offset starts near 0 with a small scale, so
    the trust region binds early and the scaling shapes the iterates: using
    x_scale in place of 1/x_scale (or ones) gives different early iterates."""
    pr = make()
    y = pr.coords()
    p0 = pr.p0.copy()
    p0[-1] = 1e-3                                   # the offset (last parameter of every model)
    xs = np.geomspace(0.5, 2.0, pr.n)
    xs[-1] = 1e-2
    for mx in (3, None):
        res = trf.fit(pr.model, y, pr.z, p0, x_scale=xs, max_nfev=mx)
        ref = least_squares(lambda x: models.h(pr.model, y, x) - pr.z, p0,
                            jac=lambda x: models.jac(pr.model, y, x), method="trf",
                            tr_solver="exact", x_scale=xs, max_nfev=mx)
        assert (res["status"], res["nfev"], res["njev"]) == (ref.status, ref.nfev, ref.njev)
        assert np.allclose(res["x"], ref.x, rtol=1e-10, atol=1e-12)
        if mx == 3 and pr.grid is None:  # (2-D: the positions dominate Delta0; the scaling does not bind)
            for other in (1.0 / xs, "ones"):
                o = trf.fit(pr.model, y, pr.z, p0, x_scale=other, max_nfev=3)
                assert not np.allclose(o["x"], res["x"], rtol=1e-6, atol=0)

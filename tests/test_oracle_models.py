"""Pins for oracle/models.py and the residual/cost definitions (Eq. 1-2).

Pinned against: complex-step derivatives (machine-exact for analytic models),
brute-force central differences (north star: 1e-7 relative on tiny inputs),
SPEC.md's trivial examples and noise-free synthesis
(r == 0 at the truth; the truth image is rendered by datagen in a different
algebraic form, so this also pins the a/b/c2 coefficients of S:463)."""
import math

import numpy as np
import pytest

import datagen as dg
from oracle import models, passes

MODELS = ["linear", "exp_decay", "gauss1d", "gauss2d_rot", "gauss2d_rot_x2"]


def _sample(model, rng, m=48):
    """Tiny random inputs: coordinates and a parameter vector in the model's
    working range."""
    if model == "linear":
        return rng.uniform(-2, 2, m), rng.uniform(-2, 2, 2)
    if model == "exp_decay":
        return rng.uniform(0, 4, m), np.array([rng.uniform(0.5, 3), rng.uniform(0.2, 2), rng.uniform(-1, 1)])
    if model == "gauss1d":
        return rng.uniform(0, 1, m), np.array([rng.uniform(0.5, 2), rng.uniform(0.3, 0.7),
                                                rng.uniform(0.05, 0.2), rng.uniform(0, 0.5)])
    W = 64
    X = rng.uniform(0, W, m)
    Y = rng.uniform(0, W, m)
    g = [rng.uniform(0.5, 2), rng.uniform(16, 48), rng.uniform(16, 48), rng.uniform(6, 16),
         rng.uniform(6, 16), rng.uniform(0, math.pi)]
    if model == "gauss2d_rot":
        return (X, Y), np.array(g + [rng.uniform(0, 0.5)])
    g2 = [rng.uniform(0.5, 2), rng.uniform(16, 48), rng.uniform(16, 48), rng.uniform(6, 16),
          rng.uniform(6, 16), rng.uniform(0, math.pi)]
    return (X, Y), np.array(g + g2 + [rng.uniform(0, 0.5)])


@pytest.mark.parametrize("model", MODELS)
def test_jacobian_matches_complex_step(model):
    rng = np.random.default_rng(101)
    for _ in range(20):
        y, x = _sample(model, rng)
        J = models.jac(model, y, x)
        n = x.size
        Jc = np.empty_like(J)
        eps = 1e-30
        for j in range(n):
            xc = x.astype(np.complex128)
            xc[j] += 1j * eps
            Jc[:, j] = np.imag(models.h(model, y, xc)) / eps
        scale = np.abs(Jc) + 1e-3 * np.max(np.abs(Jc), axis=0, keepdims=True) + 1e-300
        # analytic partials carry cancellation in a_th dx^2 + 2 b_th dx dy + c_th dy^2
        # (a_th = -c_th), so the bound is 1e-11, not eps; a wrong term is O(1)
        assert np.max(np.abs(J - Jc) / scale) < 1e-11


@pytest.mark.parametrize("model", MODELS)
def test_jacobian_matches_central_differences(model):
    """North star: analytic J vs brute-force central differences, 1e-7 relative
    (h_j = cbrt(eps) max(1, |x_j|), normalised by |J| + 1e-3 max_col |J|)."""
    rng = np.random.default_rng(202)
    y, x = _sample(model, rng, m=64)
    J = models.jac(model, y, x)
    hstep = np.cbrt(np.finfo(float).eps) * np.maximum(1.0, np.abs(x))
    Jfd = np.empty_like(J)
    for j in range(x.size):
        xp = x.copy()
        xm = x.copy()
        xp[j] += hstep[j]
        xm[j] -= hstep[j]
        Jfd[:, j] = (models.h(model, y, xp) - models.h(model, y, xm)) / (xp[j] - xm[j])
    scale = np.abs(J) + 1e-3 * np.max(np.abs(J), axis=0, keepdims=True)
    assert np.max(np.abs(J - Jfd) / scale) < 1e-7


def test_spec_trivial_examples():
    # exact model -> zero residuals; r=[3,4] -> cost 12.5
    t = np.array([1.0, 2.0, 3.0])
    r = passes.residuals("linear", t, np.array([1.0, 2.0, 3.0]), [1.0, 0.0])
    assert np.all(r == 0)
    assert passes.cost(np.array([3.0, 4.0])) == 12.5
    # linear model J = [[1,1],[2,1]] independent of x
    J1 = models.jac("linear", np.array([1.0, 2.0]), np.array([0.3, -7.0]))
    J2 = models.jac("linear", np.array([1.0, 2.0]), np.array([5.0, 2.0]))
    assert np.array_equal(J1, [[1, 1], [2, 1]]) and np.array_equal(J1, J2)


def test_gauss2d_special_values():
    # peak value A + off; isotropic at distance sx along an axis: A e^-1/2 + off
    x = np.array([1.7, 10.0, 20.0, 3.0, 3.0, 0.0, 0.25])
    X = np.array([10.0, 13.0, 10.0])
    Y = np.array([20.0, 20.0, 23.0])
    v = models.h("gauss2d_rot", (X, Y), x)
    assert v[0] == pytest.approx(1.95, abs=1e-15)
    assert v[1] == pytest.approx(1.7 * math.exp(-0.5) + 0.25, rel=1e-15)
    assert v[2] == pytest.approx(1.7 * math.exp(-0.5) + 0.25, rel=1e-15)
    # rotation by pi/2 swaps the roles of sx and sy (R22)
    xa = np.array([1.0, 5.0, 6.0, 2.0, 4.0, 0.3, 0.0])
    xb = xa.copy()
    xb[3], xb[4], xb[5] = 4.0, 2.0, 0.3 + math.pi / 2
    pts = (np.array([3.0, 7.5, 1.0]), np.array([2.0, 9.0, 6.5]))
    assert np.allclose(models.h("gauss2d_rot", pts, xa), models.h("gauss2d_rot", pts, xb), rtol=1e-14)


@pytest.mark.parametrize("make", [
    lambda: dg.make_exp_decay(noise=0.0),
    lambda: dg.make_gauss1d(500, noise=0.0),
    lambda: dg.make_gauss2d(64, noise=0.0),
    lambda: dg.make_gauss2d_x2(64, noise=0.0),
])
def test_noise_free_residual_is_zero_at_truth(make):
    pr = make()
    r = passes.residuals(pr.model, pr.coords(), pr.z, pr.truth)
    assert np.max(np.abs(r)) < 1e-12

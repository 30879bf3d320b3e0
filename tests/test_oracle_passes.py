"""Pins for oracle/passes.py (Eq. 2, 4, 5).

Pinned against brute force: pure-Python loops with math.fsum (exactly rounded
sums) over the oracle's own J rows on tiny inputs — this checks the W^T W
packing (a transposed operand or dropped term fails) — and against the
residual pass (the two passes must agree on the cost)."""
import math

import numpy as np
import pytest

import datagen as dg
from oracle import models, passes


@pytest.mark.parametrize("make", [
    lambda: dg.make_exp_decay(m=37),
    lambda: dg.make_gauss1d(41),
    lambda: dg.make_gauss2d(9),
    lambda: dg.make_gauss2d_x2(7),
])
def test_jpass_matches_fsum_brute_force(make):
    pr = make()
    y = pr.coords()
    x = pr.p0
    c, g, G, bad = passes.jpass(pr.model, y, pr.z, x)
    assert bad == 0
    J = models.jac(pr.model, y, x)
    r = models.h(pr.model, y, x) - pr.z
    n = x.size
    assert c == pytest.approx(0.5 * math.fsum(float(v) * float(v) for v in r), rel=1e-15)
    for j in range(n):
        assert g[j] == pytest.approx(math.fsum(J[i, j] * r[i] for i in range(pr.m)), rel=1e-13, abs=1e-300)
        for k in range(n):
            assert G[j, k] == pytest.approx(math.fsum(J[i, j] * J[i, k] for i in range(pr.m)), rel=1e-13)
    c2, bad2 = passes.residual_pass(pr.model, y, pr.z, x)
    assert bad2 == 0 and c2 == pytest.approx(c, rel=1e-15)


def test_nonfinite_counted():
    pr = dg.make_exp_decay(m=50)
    z = pr.z.copy()
    z[[3, 17]] = np.nan
    _, bad = passes.residual_pass(pr.model, pr.t, z, pr.p0)
    assert bad == 2
    _, _, _, bad = passes.jpass(pr.model, pr.t, z, pr.p0)
    assert bad == 2


def test_weighted_pass_equivalences():
    """App. C (Eq. C13-C16): sigma == 1 gives the unweighted pass;
    uniform sigma = s scales cost by 1/s^2, g by 1/s^2, G by 1/s^2."""
    pr = dg.make_gauss1d(300)
    y = pr.coords()
    c0, g0, G0, _ = passes.jpass(pr.model, y, pr.z, pr.p0)
    c1, g1, G1, _ = passes.jpass(pr.model, y, pr.z, pr.p0, sigma=np.ones(pr.m))
    assert c1 == c0 and np.array_equal(g1, g0) and np.array_equal(G1, G0)
    c2, g2, G2, _ = passes.jpass(pr.model, y, pr.z, pr.p0, sigma=np.full(pr.m, 2.0))
    assert c2 == pytest.approx(c0 / 4, rel=1e-14)
    assert np.allclose(g2, g0 / 4, rtol=1e-13) and np.allclose(G2, G0 / 4, rtol=1e-13)

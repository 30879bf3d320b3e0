"""Batched many-small-fits (Gpufit's regime):
jf_curve_fit_batch runs every fit of the batch in ONE launch, one warp per
fit.  Every fit must follow the oracle's trajectory (status, nfev, njev, nit
identical; x to 1e-6) — the same bar as single fits — and per-fit errors
are reported per fit."""
import numpy as np
import pytest

import datagen as dg
from oracle import trf as otrf

jf = pytest.importorskip("paper_2208_12187_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _check(res, k, ref):
    assert (res.status[k], res.nfev[k], res.njev[k], res.nit[k]) == (ref["status"], ref["nfev"], ref["njev"],
                                                                     ref["nit"]), k
    x = ref["x"]
    assert np.all(np.abs(res.x[k] - x) <= 1e-6 * np.maximum(np.abs(x), 1e-3 * np.max(np.abs(x)))), k
    assert res.cost[k] == pytest.approx(ref["cost"], rel=1e-9)


def test_batch_exp_decay_shared_t():
    probs = [dg.make_exp_decay(m=1000, k=k) for k in range(300)]
    z = np.stack([p.z for p in probs])
    res = jf.curve_fit_batch("exp_decay", z, y=probs[0].t, shared_y=True, p0=np.stack([p.p0 for p in probs]))
    for k in range(0, 300, 7):
        _check(res, k, otrf.fit("exp_decay", probs[k].t, probs[k].z, probs[k].p0))


@pytest.mark.parametrize("solver", ["auto", "gram"])
def test_batch_gauss1d_per_fit_t_device_inputs(solver):
    probs = [dg.make_gauss1d(2000, k=k) for k in range(64)]
    z = torch.as_tensor(np.stack([p.z for p in probs])).cuda()
    t = torch.as_tensor(np.stack([p.t for p in probs])).cuda()
    res = jf.curve_fit_batch("gauss1d", z, y=t, p0=np.stack([p.p0 for p in probs]), solver=solver)
    for k in range(0, 64, 3):
        _check(res, k, otrf.fit("gauss1d", probs[k].t, probs[k].z, probs[k].p0))


def test_batch_gauss2d_images_and_bounds():
    probs = [dg.make_gauss2d(32, k=k) for k in range(40)]
    z = np.stack([p.z for p in probs])
    res = jf.curve_fit_batch("gauss2d_rot", z, grid=probs[0].grid, p0=np.stack([p.p0 for p in probs]))
    for k in range(0, 40, 3):
        _check(res, k, otrf.fit("gauss2d_rot", probs[k].coords(), probs[k].z, probs[k].p0))
    pb = [dg.make_gauss2d_bounded(32, "c", k=k) for k in range(12)]
    zb = np.stack([p.z for p in pb])
    lb, ub = pb[0].lb, pb[0].ub  # shared bounds (variant c's bounds depend on the truth: use fit 0's)
    p0 = np.stack([np.clip(p.p0, lb + 1e-3, ub - 1e-3) for p in pb])
    rb = jf.curve_fit_batch("gauss2d_rot", zb, grid=pb[0].grid, p0=p0, lb=lb, ub=ub)
    for k in range(12):
        _check(rb, k, otrf.fit("gauss2d_rot", pb[k].coords(), pb[k].z, p0[k], lb, ub))


def test_batch_two_gaussians_weighted():
    probs = [dg.make_gauss2d_x2(24, k=k) for k in range(10)]
    z = np.stack([p.z for p in probs])
    sig = np.random.default_rng(4).uniform(0.5, 2.0, z.shape)
    res = jf.curve_fit_batch("gauss2d_rot_x2", z, grid=probs[0].grid, p0=np.stack([p.p0 for p in probs]), sigma=sig)
    for k in range(10):
        _check(res, k, otrf.fit("gauss2d_rot_x2", probs[k].coords(), probs[k].z, probs[k].p0, sigma=sig[k]))


def test_batch_per_fit_errors_and_default_p0():
    probs = [dg.make_exp_decay(m=500, k=k) for k in range(6)]
    z = np.stack([p.z for p in probs])
    z[2, 10] = np.nan                                  # residuals not finite at p0
    lb = np.array([0.0, 0.0, -5.0])
    ub = np.array([6.0, 4.0, 5.0])
    p0 = np.stack([p.p0 for p in probs])
    p0[4] = [7.0, 1.0, 1.0]                            # outside the bounds
    res = jf.curve_fit_batch("exp_decay", z, y=probs[0].t, shared_y=True, p0=p0, lb=lb, ub=ub)
    assert res.status[2] == -3 and res.status[4] == -2
    for k in (0, 1, 3, 5):
        _check(res, k, otrf.fit("exp_decay", probs[k].t, probs[k].z, p0[k], lb, ub))
    dflt = jf.curve_fit_batch("exp_decay", z[[0, 1]], y=probs[0].t, shared_y=True, lb=lb, ub=ub)
    for k in (0, 1):
        _check(dflt, k, otrf.fit("exp_decay", probs[k].t, probs[k].z, None, lb, ub))

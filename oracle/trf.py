"""Oracle trust-region-reflective solver.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §II step by step — Alg. 1, Alg. 2 (P:157-181,
Eq. 13-14, safeguard P:201-205), Alg. 3 with the gain
ratio Eq. 15, the scaled problem Eq. 7-8 and the SVD
solve of App. B (Eq. B1-B4) — in the paper's order.  Where the
paper is silent or at odds with itself the readings of DESIGN.md §3 apply;
they are the semantics of SciPy's TRF, which the paper names as its
algorithm ("We use SciPy's trust region method algorithm ... as the
basis", "JAXFit and SciPy use the same TRM algorithm") and whose
Coleman-Li variant JAXFit implements without detailing it (R19).

Notation: m residuals, n parameters (R1); hat quantities live in the scaled
space p = D w (Eq. 8); d = diag(D^{-1}); J_h = J diag(d); g_h = d * g.
"""
from __future__ import annotations

import math

import numpy as np

from . import models

EPS = np.finfo(np.float64).eps


# ---------------------------------------------------------------------------
# Alg. 2 + App. B: the Levenberg-Marquardt parameter and the step
# ---------------------------------------------------------------------------

def phi_and_derivative(alpha, suf, s, Delta):
    """Eq. 13 in the SVD basis (Eq. B4): p(alpha) = -V (S^T S + alpha)^-1 S^T U^T r,
    so ||p|| = ||suf / (s^2 + alpha)||, phi = ||p|| - Delta, and (reading R11)
    phi' = -sum(suf^2 / (s^2+alpha)^3) / ||p||."""
    denom = s * s + alpha
    q = suf / denom
    pn = float(np.linalg.norm(q))
    phi = pn - Delta
    dphi = -float(np.sum(suf * suf / denom**3)) / pn
    return phi, dphi


def solve_tr(n, m, uf, s, V, Delta, alpha):
    """Alg. 1 lines 141-148 and Alg. 2, in the SVD basis of App. B.

    uf = U^T r, s = singular values (descending), V (columns = right singular
    vectors) of the scaled Jacobian.  Returns (p, alpha, n_iter); n_iter == 0
    means the Gauss-Newton trial p_t = -B^-1 g was accepted.

    Readings: R5 (alpha warm start), R6 (rank test s_min > EPS m s_max before
    the Gauss-Newton trial), R7/R8 (p = -(B + alpha I)^-1 g), R9 (iterate
    until |phi| < sigma Delta, sigma = 0.01, at most 10 iterations), R10 (the
    order of the safeguard, the u / l updates and the Newton step Eq. 14),
    R12 (final p scaled to ||p|| = Delta)."""
    suf = s * uf
    full_rank = (m >= n) and (s[-1] > EPS * m * s[0])
    if full_rank:
        p = -V.dot(uf / s)                       # Alg. 1 l.141: p_t = -B^-1 g (Eq. B4, alpha=0)
        if np.linalg.norm(p) <= Delta:           # Alg. 1 l.142
            return p, 0.0, 0
    u = float(np.linalg.norm(suf)) / Delta       # Alg. 2 l.160: u = ||g_hat|| / Delta
    if full_rank:
        phi, dphi = phi_and_derivative(0.0, suf, s, Delta)
        l = -phi / dphi                          # Alg. 2 l.161
    else:
        l = 0.0
    if not full_rank and alpha == 0:
        alpha = max(0.001 * u, math.sqrt(l * u))
    it = 0
    for it in range(10):                         # R9: cap 10
        if alpha < l or alpha > u:               # P:201-203 safeguard
            alpha = max(0.001 * u, math.sqrt(l * u))
        phi, dphi = phi_and_derivative(alpha, suf, s, Delta)
        if phi < 0:                              # Alg. 2 l.173-175
            u = alpha
        ratio = phi / dphi
        l = max(l, alpha - ratio)                # Alg. 2 l.172
        alpha = alpha - ((phi + Delta) / Delta) * ratio   # Eq. 14
        if abs(phi) < 0.01 * Delta:              # R9: sigma = 0.01, strict
            break
    p = -V.dot(suf / (s * s + alpha))            # Eq. B4 (sign R8)
    p = p * (Delta / np.linalg.norm(p))          # R12
    return p, alpha, it + 1


# ---------------------------------------------------------------------------
# Alg. 3 and Eq. 15 (reading R14, R15), termination (R16)
# ---------------------------------------------------------------------------

def update_radius(Delta, actual, predicted, step_norm, bound_hit):
    """Eq. 15 gain ratio and the radius update of Alg. 3 with SciPy's rules.

    gamma = actual / predicted if predicted > 0; 1 if both are 0; else 0 (R14).
    gamma < 0.25 -> Delta = 0.25 ||p_h||; gamma > 0.75 and ||p_h|| > 0.95 Delta
    -> Delta = 2 Delta; otherwise unchanged (R15)."""
    if predicted > 0:
        ratio = actual / predicted
    elif predicted == 0 and actual == 0:
        ratio = 1.0
    else:
        ratio = 0.0
    if ratio < 0.25:
        Delta = 0.25 * step_norm
    elif ratio > 0.75 and bound_hit:
        Delta = 2.0 * Delta
    return Delta, ratio


def termination(dF, F, dx_norm, x_norm, ratio, ftol, xtol):
    """The 'accuracy condition' of Alg. 1 l.139 (reading R16).  Returns the
    status 4 (ftol and xtol), 2 (ftol), 3 (xtol) or None."""
    ftol_ok = dF < ftol * F and ratio > 0.25
    xtol_ok = dx_norm < xtol * (xtol + x_norm)
    if ftol_ok and xtol_ok:
        return 4
    if ftol_ok:
        return 2
    if xtol_ok:
        return 3
    return None


def jac_scale(J, scale_inv_old=None):
    """Reading R3: D = diag(column norms of J), running max over iterations,
    zero columns -> 1 at the first iteration.  Returns scale_inv = diag(D)."""
    si = np.sqrt(np.sum(J * J, axis=0))
    if scale_inv_old is None:
        si[si == 0] = 1.0
    else:
        si = np.maximum(si, scale_inv_old)
    return si


# ---------------------------------------------------------------------------
# Coleman-Li machinery (reading R19, R20)
# ---------------------------------------------------------------------------

def cl_vector(x, g, lb, ub):
    """Coleman-Li scaling vector v and its derivative dv."""
    v = np.ones_like(x)
    dv = np.zeros_like(x)
    msk = (g < 0) & np.isfinite(ub)
    v[msk] = ub[msk] - x[msk]
    dv[msk] = -1.0
    msk = (g > 0) & np.isfinite(lb)
    v[msk] = x[msk] - lb[msk]
    dv[msk] = 1.0
    return v, dv


def active_set(x, lb, ub, rtol):
    """-1 / +1 where a lower / upper bound is active (relative tolerance rtol)."""
    act = np.zeros(x.shape, dtype=np.int64)
    if rtol == 0:
        act[x <= lb] = -1
        act[x >= ub] = 1
        return act
    ld = x - lb
    ud = ub - x
    lt = rtol * np.maximum(1.0, np.abs(lb))
    ut = rtol * np.maximum(1.0, np.abs(ub))
    lo = np.isfinite(lb) & (ld <= np.minimum(ud, lt))
    act[lo] = -1
    up = np.isfinite(ub) & (ud <= np.minimum(ld, ut))
    act[up] = 1
    return act


def strictly_feasible(x, lb, ub, rstep):
    """Move x into the interior: rstep = 0 -> the next float towards the other
    bound; else bound +- rstep*max(1,|bound|); still outside -> midpoint."""
    xn = x.copy()
    act = active_set(x, lb, ub, rstep)
    lo = act == -1
    up = act == 1
    if rstep == 0:
        xn[lo] = np.nextafter(lb[lo], ub[lo])
        xn[up] = np.nextafter(ub[up], lb[up])
    else:
        xn[lo] = lb[lo] + rstep * np.maximum(1.0, np.abs(lb[lo]))
        xn[up] = ub[up] - rstep * np.maximum(1.0, np.abs(ub[up]))
    tight = (xn < lb) | (xn > ub)
    xn[tight] = 0.5 * (lb[tight] + ub[tight])
    return xn


def step_to_bound(x, s, lb, ub):
    """Smallest t >= 0 with x + t s on a bound, and the hit pattern
    (sign(s_j) for every j attaining the minimum, R20)."""
    steps = np.full(x.shape, np.inf)
    nz = s != 0
    with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
        steps[nz] = np.maximum((lb - x)[nz] / s[nz], (ub - x)[nz] / s[nz])
    t = float(np.min(steps))
    hits = (steps == t).astype(np.int64) * np.sign(s).astype(np.int64)
    return t, hits


def tr_intersect(x, s, Delta):
    """Roots t of ||x + t s|| = Delta (stable form), returned (t_neg, t_pos)."""
    a = float(np.dot(s, s))
    b = float(np.dot(x, s))
    c = float(np.dot(x, x)) - Delta * Delta
    d = math.sqrt(b * b - a * c)
    q = -(b + math.copysign(d, b))
    t1 = q / a
    t2 = c / q
    return (t1, t2) if t1 < t2 else (t2, t1)


def quad_1d(Jh, gh, s, diag=None, s0=None):
    """Coefficients of Q(s0 + t s) = a t^2 + b t + c, where
    Q(w) = 1/2 w^T (J_h^T J_h + diag) w + g_h^T w (the model of Eq. 6 in hat space)."""
    v = Jh.dot(s)
    a = float(np.dot(v, v))
    if diag is not None:
        a += float(np.dot(s * diag, s))
    a *= 0.5
    b = float(np.dot(gh, s))
    if s0 is None:
        return a, b, 0.0
    u = Jh.dot(s0)
    b += float(np.dot(u, v))
    c = 0.5 * float(np.dot(u, u)) + float(np.dot(gh, s0))
    if diag is not None:
        b += float(np.dot(s0 * diag, s))
        c += 0.5 * float(np.dot(s0 * diag, s0))
    return a, b, c


def min_quad_1d(a, b, lo, hi, c=0.0):
    """Minimise a t^2 + b t + c on [lo, hi]: candidates lo, hi, then the vertex
    if strictly inside; the first minimiser wins (R20)."""
    ts = [lo, hi]
    if a != 0:
        ext = -0.5 * b / a
        if lo < ext < hi:
            ts.append(ext)
    ys = [t * (a * t + b) + c for t in ts]
    k = int(np.argmin(ys))
    return ts[k], ys[k]


def eval_quad(Jh, gh, s, diag=None):
    """Q(s) = 1/2 (||J_h s||^2 + s^T diag s) + g_h^T s (Eq. 6 in hat space, R13)."""
    Js = Jh.dot(s)
    q = float(np.dot(Js, Js))
    if diag is not None:
        q += float(np.dot(s * diag, s))
    return 0.5 * q + float(np.dot(s, gh))


def select_step(x, Jh, diag_h, gh, p, p_h, d, Delta, lb, ub, theta):
    """Coleman-Li step selection (R19, R20): the full step if it stays feasible;
    otherwise the best of the theta-truncated step, the reflected step and the
    scaled (anti)gradient.  Returns (step, step_h, predicted_reduction, branch),
    branch 0 interior, 1 reflected, 2 truncated, 3 gradient."""
    if np.all((x + p >= lb) & (x + p <= ub)):
        return p, p_h, -eval_quad(Jh, gh, p_h, diag_h), 0
    t_b, hits = step_to_bound(x, p, lb, ub)
    r_h = p_h.copy()
    r_h[hits.astype(bool)] *= -1
    r = d * r_h
    p = p * t_b
    p_h = p_h * t_b
    x_b = x + p
    _, to_tr = tr_intersect(p_h, r_h, Delta)
    to_bd, _ = step_to_bound(x_b, r, lb, ub)
    rs = min(to_bd, to_tr)
    if rs > 0:
        lo = (1 - theta) * t_b / rs
        hi = theta * to_bd if rs == to_bd else to_tr
    else:
        lo, hi = 0.0, -1.0
    if lo <= hi:
        a, b, c = quad_1d(Jh, gh, r_h, diag_h, p_h)
        rt, r_val = min_quad_1d(a, b, lo, hi, c)
        r_h = p_h + rt * r_h
        r = r_h * d
    else:
        r_val = np.inf
    p = p * theta
    p_h = p_h * theta
    p_val = eval_quad(Jh, gh, p_h, diag_h)
    ag_h = -gh
    ag = d * ag_h
    t_tr = Delta / np.linalg.norm(ag_h)
    t_bd, _ = step_to_bound(x, ag, lb, ub)
    stride = theta * t_bd if t_bd < t_tr else t_tr
    a, b, _ = quad_1d(Jh, gh, ag_h, diag_h)
    at, ag_val = min_quad_1d(a, b, 0.0, stride)
    ag_h = ag_h * at
    ag = ag * at
    if p_val < r_val and p_val < ag_val:
        return p, p_h, -p_val, 2
    if r_val < p_val and r_val < ag_val:
        return r, r_h, -r_val, 1
    return ag, ag_h, -ag_val, 3


# ---------------------------------------------------------------------------
# Alg. 1: the fit
# ---------------------------------------------------------------------------

class FitError(ValueError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def default_p0(n, lb, ub):
    """curve_fit's default initial guess (reading for p0 = NULL in jf.h)."""
    p0 = np.ones(n)
    lf = np.isfinite(lb)
    uf = np.isfinite(ub)
    both = lf & uf
    p0[both] = 0.5 * (lb[both] + ub[both])
    p0[lf & ~uf] = lb[lf & ~uf] + 1
    p0[~lf & uf] = ub[~lf & uf] - 1
    return p0


def fit(model, y, z, p0=None, lb=None, ub=None, ftol=1e-8, xtol=1e-8, gtol=1e-8,
        max_nfev=None, x_scale="jac", sigma=None, trace=None):
    """Alg. 1 with Alg. 2, Alg. 3, Eq. 15 and App. B.

    model: oracle model name; y: t or (X, Y); z: observations.  x_scale:
    'jac', 'ones' or an array (R3).  sigma: optional per-point errors
    (App. C diagonal case, Eq. C13-C16).  trace: optional list receiving one
    record per trial (see jf.h JF_TRACE_FIELDS).

    Returns dict(x, cost, grad, gram, optimality, status, nfev, njev, nit,
    active_mask).  Raises FitError(code) on invalid input (R18)."""
    n = models.NPARAMS[model]
    z = np.asarray(z, dtype=np.float64)
    m = z.shape[0]
    lb = np.full(n, -np.inf) if lb is None else np.asarray(lb, dtype=np.float64).copy()
    ub = np.full(n, np.inf) if ub is None else np.asarray(ub, dtype=np.float64).copy()
    if np.any(np.isnan(lb)) or np.any(np.isnan(ub)) or np.any(lb >= ub):
        raise FitError(-1, "each lower bound must be strictly less than its upper bound")
    bounded = bool(np.any(np.isfinite(lb)) or np.any(np.isfinite(ub)))
    x = default_p0(n, lb, ub) if p0 is None else np.asarray(p0, dtype=np.float64).copy()
    if np.any(x < lb) or np.any(x > ub):
        raise FitError(-2, "p0 is infeasible")
    if max_nfev is None or max_nfev == 0:
        max_nfev = 100 * n
    if bounded:
        x = strictly_feasible(x, lb, ub, 1e-10)

    w = None if sigma is None else 1.0 / np.asarray(sigma, dtype=np.float64)

    def fun(xv):                                   # Eq. 1 (weighted: Eq. C16)
        r = models.h(model, y, xv) - z
        return r if w is None else r * w

    def jacf(xv):                                  # P:66-75 (weighted: Eq. C15)
        J = models.jac(model, y, xv)
        return J if w is None else J * w[:, None]

    f = fun(x)
    if not np.all(np.isfinite(f)):
        raise FitError(-3, "residuals are not finite at the initial point")
    nfev = 1
    J = jacf(x)
    njev = 1
    cost = 0.5 * float(np.dot(f, f))             # Eq. 2
    g = J.T.dot(f)                                # Eq. 4

    if isinstance(x_scale, str) and x_scale == "jac":
        scale_inv = jac_scale(J)
        jacmode = True
    else:
        xs = np.ones(n) if (isinstance(x_scale, str) and x_scale == "ones") else np.asarray(x_scale, float)
        scale_inv = 1.0 / xs
        jacmode = False

    if bounded:                                   # R4
        v, dv = cl_vector(x, g, lb, ub)
        v[dv != 0] *= scale_inv[dv != 0]
        Delta = float(np.linalg.norm(x * scale_inv / np.sqrt(v)))
    else:
        Delta = float(np.linalg.norm(x * scale_inv))
    if Delta == 0:
        Delta = 1.0

    alpha = 0.0
    status = None
    nit = 0
    gnorm = 0.0
    while True:
        if bounded:
            v, dv = cl_vector(x, g, lb, ub)
            gnorm = float(np.linalg.norm(g * v, ord=np.inf))
        else:
            gnorm = float(np.linalg.norm(g, ord=np.inf))
        if gnorm < gtol:                          # R16 (gtol)
            status = 1
        if status is not None or nfev == max_nfev:
            break

        if bounded:                               # R19: Coleman-Li hat space
            v[dv != 0] *= scale_inv[dv != 0]
            d = np.sqrt(v) / scale_inv
            diag_h = g * dv / scale_inv
        else:                                     # Eq. 8: J_hat = J D^-1
            d = 1.0 / scale_inv
            diag_h = None
        g_h = d * g
        J_h = J * d
        if bounded:                               # App. B on [J_h; diag(sqrt(diag_h))]
            Jaug = np.vstack([J_h, np.diag(np.sqrt(diag_h))])
            faug = np.concatenate([f, np.zeros(n)])
            U, s, VT = np.linalg.svd(Jaug, full_matrices=False)
            uf = U.T.dot(faug)
            theta = max(0.995, 1.0 - gnorm)
        else:                                     # App. B: J_h = U S V^T
            U, s, VT = np.linalg.svd(J_h, full_matrices=False)
            uf = U.T.dot(f)
        V = VT.T

        actual = -1.0
        while actual <= 0 and nfev < max_nfev:    # R15: retry with the same SVD
            Delta_used = Delta
            p_h, alpha, _ = solve_tr(n, m, uf, s, V, Delta, alpha)
            if bounded:
                p = d * p_h
                step, step_h, pred, branch = select_step(x, J_h, diag_h, g_h, p, p_h, d, Delta, lb, ub, theta)
                x_new = strictly_feasible(x + step, lb, ub, 0.0)
            else:
                step_h = p_h
                pred = -eval_quad(J_h, g_h, step_h)      # Eq. 15 denominator (R13)
                step = d * step_h                        # Alg. 3 l.185: w = D^-1 p
                x_new = x + step
                branch = -1
            f_new = fun(x_new)
            nfev += 1
            hn = float(np.linalg.norm(step_h))
            if not np.all(np.isfinite(f_new)):   # R17
                Delta = 0.25 * hn
                if trace is not None:
                    trace.append([nit, nfev, njev, cost, math.nan, Delta_used, alpha, math.nan,
                                  hn, float(np.linalg.norm(step)), pred, branch])
                continue
            cost_new = 0.5 * float(np.dot(f_new, f_new))
            actual = cost - cost_new
            Delta_new, ratio = update_radius(Delta, actual, pred, hn, hn > 0.95 * Delta)
            step_norm = float(np.linalg.norm(step))
            if trace is not None:
                trace.append([nit, nfev, njev, cost, cost_new, Delta_used, alpha, ratio,
                              hn, step_norm, pred, branch])
            status = termination(actual, cost, step_norm, float(np.linalg.norm(x)), ratio, ftol, xtol)
            if status is not None:
                break
            alpha *= Delta / Delta_new                   # R5
            Delta = Delta_new

        if actual > 0:                            # accepted (R15)
            x = x_new
            f = f_new
            cost = cost_new
            J = jacf(x)
            njev += 1
            g = J.T.dot(f)
            if jacmode:
                scale_inv = jac_scale(J, scale_inv)
        nit += 1                                  # R27

    if status is None:
        status = 0
    act = active_set(x, lb, ub, xtol) if bounded else np.zeros(n, dtype=np.int64)
    return dict(x=x, cost=cost, grad=g, gram=J.T.dot(J), optimality=gnorm, status=status,
                nfev=nfev, njev=njev, nit=nit, active_mask=act, m=m, n=n, pcov=pcov(J, cost))


def pcov(J, cost):
    """Parameter covariance as curve_fit returns it with the fit (reading for
    SURVEY A29 / N3): Moore-Penrose inverse of J^T J through the SVD of J,
    singular values <= EPS max(m, n) s_max discarded, scaled by the residual
    variance 2 cost / (m - n) (m > n; else +inf)."""
    m, n = J.shape
    _, s, VT = np.linalg.svd(J, full_matrices=False)
    keep = s > EPS * max(m, n) * s[0]
    s = s[keep]
    VT = VT[: s.size]
    P = (VT.T / s**2).dot(VT)
    if m > n:
        return P * (2.0 * cost / (m - n))
    return np.full((n, n), np.inf)

"""Oracle per-pass quantities.  TEST INFRASTRUCTURE ONLY.

  residuals  r_i = h(y_i; x) - z_i                    P:45-48 Eq. 1
  cost       f = 1/2 r^T r                             P:50-53 Eq. 2
  gradient   g = J^T r                                 P:61-65 Eq. 4
  Gram       B = J^T J (Gauss-Newton Hessian)          P:76-81 Eq. 5

The J-pass of the CUDA path reduces the upper triangle of W^T W with
W = [J | r] (cost = slot(n,n)/2, g = column n, G = the n x n block); the
oracle forms J explicitly (as App. B does), builds W, and takes W^T W with a
matrix product in extended precision (numpy longdouble, x87 80-bit on this
host), so the oracle's own rounding is far below the 1e-10 parity tolerance
(reading R24).  Rows are processed in chunks only to bound memory; the sum
over i is the definition's, order-free in exact arithmetic.
"""
from __future__ import annotations

import numpy as np

from . import models

CHUNK = 1 << 20


def _slice_y(y, lo, hi):
    if isinstance(y, tuple):
        return tuple(c[lo:hi] for c in y)
    return y[lo:hi]


def residuals(model, y, z, x):
    """Eq. 1: r_i = h(y_i; x) - z_i."""
    return models.h(model, y, np.asarray(x, dtype=np.float64)) - z


def cost(r):
    """Eq. 2: f = 1/2 sum r_i^2, accumulated in extended precision."""
    rl = np.asarray(r, dtype=np.longdouble)
    return float(0.5 * np.dot(rl, rl))


def residual_pass(model, y, z, x, sigma=None):
    """Residual-only pass: (cost, nonfinite count) at x (Eq. 1-2; R17).
    When the count is non-zero the cost is not finite (its value is unspecified).

    With sigma (App. C, P:346-352 Eq. C1; reading R25), r~_i = r_i / sigma_i."""
    m = z.shape[0]
    acc = np.longdouble(0)
    bad = 0
    for lo in range(0, m, CHUNK):
        hi = min(m, lo + CHUNK)
        r = residuals(model, _slice_y(y, lo, hi), z[lo:hi], x)
        if sigma is not None:
            r = r / sigma[lo:hi]
        bad += int((~np.isfinite(r)).sum())
        rl = r.astype(np.longdouble)
        acc += np.dot(rl, rl)
    return float(0.5 * acc), bad


def jpass(model, y, z, x, sigma=None):
    """J-pass: (cost, g, G, nonfinite) at x — Eq. 2, 4, 5 with J materialised.

    With sigma: J~ = diag(1/sigma) J, r~ = r / sigma (P:418-422 Eq. C13-C14)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.size
    m = z.shape[0]
    WtW = np.zeros((n + 1, n + 1), dtype=np.longdouble)
    bad = 0
    for lo in range(0, m, CHUNK):
        hi = min(m, lo + CHUNK)
        ys = _slice_y(y, lo, hi)
        r = residuals(model, ys, z[lo:hi], x)
        J = models.jac(model, ys, x)
        if sigma is not None:
            w = 1.0 / sigma[lo:hi]
            r = r * w
            J = J * w[:, None]
        bad += int((~np.isfinite(r)).sum())
        W = np.concatenate([J, r[:, None]], axis=1).astype(np.longdouble)
        WtW += W.T @ W
    G = np.array(WtW[:n, :n], dtype=np.float64)
    g = np.array(WtW[:n, n], dtype=np.float64)
    c = float(0.5 * WtW[n, n])
    return c, g, G, bad

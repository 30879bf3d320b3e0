"""Oracle models h(y; x) and hand-derived analytic Jacobians.  TEST INFRASTRUCTURE ONLY.

P:44-48 §II Eq. 1 defines r_i(x) = h(y_i, x) - z_i; the Jacobian J
is dr_i/dx_j = dh(y_i; x)/dx_j.  The paper computes J by autodiff;
the oracle instead uses the closed-form partials below (the north star's
"finite-difference-checked analytic Jacobians"), so that the CUDA path's
forward-mode dual numbers and the oracle are two independent derivations.

Every function accepts complex parameter vectors so tests can pin the
partials by the complex-step derivative Im h(x + i eps e_j) / eps.

Parameter orders (reading R21; SPEC.md S:463 for the 2-D form):
  linear          (x0, x1)                 h = x0 t + x1
  exp_decay       (a, b, c)                h = a exp(-b t) + c
  gauss1d         (A, mu, s, c)            h = A exp(-(t-mu)^2/(2 s^2)) + c
  gauss2d_rot     (A, x0, y0, sx, sy, th, off)
                  h = A exp(-(a dx^2 + 2 b dx dy + c2 dy^2)) + off,  dx = X-x0, dy = Y-y0
                  a  = cos^2/(2 sx^2) + sin^2/(2 sy^2)
                  b  = sin(2th) (1/(4 sy^2) - 1/(4 sx^2))
                  c2 = sin^2/(2 sx^2) + cos^2/(2 sy^2)
  gauss2d_rot_x2  (A1,x1,y1,sx1,sy1,th1, A2,x2,y2,sx2,sy2,th2, off)
                  two gauss2d_rot without offsets plus one shared offset
"""
from __future__ import annotations

import numpy as np

NPARAMS = {"linear": 2, "exp_decay": 3, "gauss1d": 4, "gauss2d_rot": 7, "gauss2d_rot_x2": 13}
YDIM = {"linear": 1, "exp_decay": 1, "gauss1d": 1, "gauss2d_rot": 2, "gauss2d_rot_x2": 2}


def _shape_coeffs(sx, sy, th):
    """a, b, c2 of the rotated Gaussian and their partials w.r.t. (sx, sy, th)."""
    C = np.cos(th)
    S = np.sin(th)
    S2 = np.sin(2 * th)
    C2 = np.cos(2 * th)
    a = C * C / (2 * sx * sx) + S * S / (2 * sy * sy)
    b = S2 * (1 / (4 * sy * sy) - 1 / (4 * sx * sx))
    c = S * S / (2 * sx * sx) + C * C / (2 * sy * sy)
    a_sx = -C * C / sx**3
    a_sy = -S * S / sy**3
    a_th = S2 * (1 / (2 * sy * sy) - 1 / (2 * sx * sx))
    b_sx = S2 / (2 * sx**3)
    b_sy = -S2 / (2 * sy**3)
    b_th = C2 * (1 / (2 * sy * sy) - 1 / (2 * sx * sx))
    c_sx = -S * S / sx**3
    c_sy = -C * C / sy**3
    c_th = -a_th
    return (a, b, c), (a_sx, b_sx, c_sx), (a_sy, b_sy, c_sy), (a_th, b_th, c_th)


def _gauss2d_value_and_cols(X, Y, A, x0, y0, sx, sy, th):
    """Value A*E and the six partials w.r.t. (A, x0, y0, sx, sy, th)."""
    (a, b, c), dsx, dsy, dth = _shape_coeffs(sx, sy, th)
    dx = X - x0
    dy = Y - y0
    q = a * dx * dx + 2 * b * dx * dy + c * dy * dy
    E = np.exp(-q)
    AE = A * E

    def dq(coef):
        ca, cb, cc = coef
        return ca * dx * dx + 2 * cb * dx * dy + cc * dy * dy

    cols = [
        E,                                   # d/dA
        AE * (2 * a * dx + 2 * b * dy),      # d/dx0
        AE * (2 * b * dx + 2 * c * dy),      # d/dy0
        -AE * dq(dsx),                       # d/dsx
        -AE * dq(dsy),                       # d/dsy
        -AE * dq(dth),                       # d/dth
    ]
    return AE, cols


def h(model: str, y, x):
    """Model value h(y; x) (Eq. 1's h).  y: t (1-D) or (X, Y) (2-D)."""
    if model == "linear":
        return x[0] * y + x[1]
    if model == "exp_decay":
        return x[0] * np.exp(-x[1] * y) + x[2]
    if model == "gauss1d":
        A, mu, s, c = x
        d = y - mu
        return A * np.exp(-d * d / (2 * s * s)) + c
    X, Y = y
    if model == "gauss2d_rot":
        v, _ = _gauss2d_value_and_cols(X, Y, *x[0:6])
        return v + x[6]
    if model == "gauss2d_rot_x2":
        v1, _ = _gauss2d_value_and_cols(X, Y, *x[0:6])
        v2, _ = _gauss2d_value_and_cols(X, Y, *x[6:12])
        return v1 + v2 + x[12]
    raise ValueError(f"unknown model {model!r}")


def jac(model: str, y, x):
    """Analytic Jacobian dh/dx, shape (m, n)."""
    if model == "linear":
        t = np.asarray(y)
        return np.stack([t, np.ones_like(t)], axis=1)
    if model == "exp_decay":
        a, b, _ = x
        t = np.asarray(y)
        E = np.exp(-b * t)
        return np.stack([E, -a * t * E, np.ones_like(E)], axis=1)
    if model == "gauss1d":
        A, mu, s, _ = x
        t = np.asarray(y)
        d = t - mu
        E = np.exp(-d * d / (2 * s * s))
        AE = A * E
        return np.stack([E, AE * d / (s * s), AE * d * d / s**3, np.ones_like(E)], axis=1)
    X, Y = y
    if model == "gauss2d_rot":
        _, cols = _gauss2d_value_and_cols(X, Y, *x[0:6])
        return np.stack(cols + [np.ones_like(cols[0])], axis=1)
    if model == "gauss2d_rot_x2":
        _, c1 = _gauss2d_value_and_cols(X, Y, *x[0:6])
        _, c2 = _gauss2d_value_and_cols(X, Y, *x[6:12])
        return np.stack(c1 + c2 + [np.ones_like(c1[0])], axis=1)
    raise ValueError(f"unknown model {model!r}")

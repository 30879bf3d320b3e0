"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module is the ONLY code both sides of a parity comparison use.  It holds
no arithmetic of the method (no residual, Jacobian, reduction or solver step):
it draws parameters and noise and synthesises observations z = h(y; truth) +
noise, where the truth images are rendered with the model written in its own
geometric form (rotated coordinates u, v below) rather than the a/b/c2
coefficient form the oracle and the CUDA kernels evaluate.

Workloads follow PAPER.md §IV: 2D rotated elliptical Gaussians with
seven parameters drawn uniformly, additive zero-mean Gaussian noise of fixed
standard deviation, data lengths log-spaced in [1e4, 8e6].  The paper states
neither the parameter ranges nor the noise level; the ranges are SPEC.md's
 and the recipe is SURVEY.md §8(d) d.2 (listed in DESIGN.md §4).

RNG call order (fixed so every consumer sees identical bytes):
    rng   = numpy.random.default_rng([seed, k])       # k = image index in the config
    truth = [rng.uniform(lo_j, hi_j) for j in parameter order]
    delta = rng.uniform(-dp, dp, n)                   # dp = 0.2 (0.1 for C5)
    p0    = truth * (1 + delta); theta params: truth + delta (absolute radians)
    noise = sigma_n * rng.standard_normal(m)          # pixel i = row*W + col
    z     = h(y; truth) + noise
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Model names and parameter counts (the problem statement, P:44 and R21).
MODELS = {
    "linear": (2, 1),
    "exp_decay": (3, 1),
    "gauss1d": (4, 1),
    "gauss2d_rot": (7, 2),
    "gauss2d_rot_x2": (13, 2),
}

# Indices of rotation-angle parameters (their p0 perturbation is absolute).
THETA_PARAMS = {"gauss2d_rot": (5,), "gauss2d_rot_x2": (5, 11)}


@dataclass
class Problem:
    """One synthetic fit problem.

    model: a key of MODELS.  z: observations (float64, length m).
    t: explicit 1-D abscissae (1-D models) or None.
    grid: (W, H, row0) for image models: point i is pixel (row=i//W, col=i%W),
          X = col, Y = row + row0 (reading R21).
    truth, p0: float64 parameter vectors.  lb/ub: bounds or None.
    """

    model: str
    z: np.ndarray
    truth: np.ndarray
    p0: np.ndarray
    t: np.ndarray | None = None
    grid: tuple[int, int, int] | None = None
    lb: np.ndarray | None = None
    ub: np.ndarray | None = None
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.z.shape[0])

    @property
    def n(self) -> int:
        return MODELS[self.model][0]

    def coords(self):
        """Explicit independent variables: t (1-D) or (X, Y) (2-D), float64."""
        if self.grid is None:
            return self.t
        return grid_coords(*self.grid)


def grid_coords(W: int, H: int, row0: int = 0):
    """Pixel-centre coordinates of a W x H row-major grid (reading R21)."""
    cols = np.arange(W, dtype=np.float64)
    rows = np.arange(row0, row0 + H, dtype=np.float64)
    X = np.broadcast_to(cols[None, :], (H, W)).reshape(-1).copy()
    Y = np.broadcast_to(rows[:, None], (H, W)).reshape(-1).copy()
    return X, Y


# ---------------------------------------------------------------------------
# Rendering of the truth (data synthesis only; written in geometric form).
# ---------------------------------------------------------------------------

def _render_gauss2d(X, Y, A, x0, y0, sx, sy, th):
    # Rotated frame: u along the sx axis, v along the sy axis.  This form is
    # algebraically equal to A*exp(-(a dx^2 + 2b dx dy + c2 dy^2)) with SPEC
    # S:463's a, b, c2 (their b = sin2t (1/(4sy^2) - 1/(4sx^2)) fixes the
    # rotation sense below).
    dx = X - x0
    dy = Y - y0
    u = math.cos(th) * dx - math.sin(th) * dy
    v = math.sin(th) * dx + math.cos(th) * dy
    return A * np.exp(-0.5 * ((u / sx) ** 2 + (v / sy) ** 2))


def render(model: str, coords, p) -> np.ndarray:
    """h(y; p) for synthesis of observations."""
    p = [float(v) for v in p]
    if model == "linear":
        return p[0] * coords + p[1]
    if model == "exp_decay":
        return p[0] * np.exp(-p[1] * coords) + p[2]
    if model == "gauss1d":
        A, mu, s, c = p
        return A * np.exp(-0.5 * ((coords - mu) / s) ** 2) + c
    X, Y = coords
    if model == "gauss2d_rot":
        return _render_gauss2d(X, Y, *p[:6]) + p[6]
    if model == "gauss2d_rot_x2":
        return _render_gauss2d(X, Y, *p[0:6]) + _render_gauss2d(X, Y, *p[6:12]) + p[12]
    raise ValueError(model)


# ---------------------------------------------------------------------------
# Configurations (BASELINE.json configs)
# ---------------------------------------------------------------------------

def _ranges_gauss2d(W: int):
    return [
        (0.5, 2.0),                 # A
        (W / 4, 3 * W / 4),         # x0
        (W / 4, 3 * W / 4),         # y0
        (W / 10, W / 4),            # sx
        (W / 10, W / 4),            # sy
        (0.0, math.pi),             # theta
        (0.0, 0.5),                 # off
    ]


def _ranges_gauss2d_x2(W: int):
    g1 = [(0.5, 2.0), (W / 5, 2 * W / 5), (W / 4, 3 * W / 4), (W / 20, W / 8), (W / 20, W / 8), (0.0, math.pi)]
    g2 = [(0.5, 2.0), (3 * W / 5, 4 * W / 5), (W / 4, 3 * W / 4), (W / 20, W / 8), (W / 20, W / 8), (0.0, math.pi)]
    return g1 + g2 + [(0.0, 0.5)]


def _draw(rng, ranges, model, dp):
    truth = np.array([rng.uniform(lo, hi) for lo, hi in ranges], dtype=np.float64)
    n = truth.size
    delta = rng.uniform(-dp, dp, n)
    p0 = truth * (1.0 + delta)
    for j in THETA_PARAMS.get(model, ()):
        p0[j] = truth[j] + delta[j]
    return truth, p0


def make_exp_decay(m: int = 1000, seed: int = 1, k: int = 0, noise: float = 0.2) -> Problem:
    """C1: a*exp(-b t)+c, t_i = 4 i/(m-1), truth (2.5, 1.3, 0.5), p0 = ones."""
    rng = np.random.default_rng([seed, k])
    t = 4.0 * np.arange(m, dtype=np.float64) / (m - 1)
    truth = np.array([2.5, 1.3, 0.5])
    z = render("exp_decay", t, truth) + noise * rng.standard_normal(m)
    return Problem("exp_decay", z, truth, np.ones(3), t=t, name=f"C1 m={m}")


def make_gauss1d(m: int, seed: int = 2, k: int = 0, noise: float = 0.05) -> Problem:
    """C2: A exp(-(t-mu)^2/(2 s^2)) + c, t_i = i/m."""
    rng = np.random.default_rng([seed, k])
    ranges = [(0.5, 2.0), (0.3, 0.7), (0.03, 0.1), (0.0, 0.5)]
    truth, p0 = _draw(rng, ranges, "gauss1d", 0.2)
    t = np.arange(m, dtype=np.float64) / m
    z = render("gauss1d", t, truth) + noise * rng.standard_normal(m)
    return Problem("gauss1d", z, truth, p0, t=t, name=f"C2 m={m}", meta={"t0": 0.0, "dt": 1.0 / m})


def make_gauss2d(W: int, seed: int = 3, k: int = 0, noise: float = 0.1, H: int | None = None) -> Problem:
    """C3 / T: rotated 2D Gaussian + offset on a W x H implicit grid."""
    H = W if H is None else H
    rng = np.random.default_rng([seed, k])
    truth, p0 = _draw(rng, _ranges_gauss2d(W), "gauss2d_rot", 0.2)
    X, Y = grid_coords(W, H)
    z = render("gauss2d_rot", (X, Y), truth) + noise * rng.standard_normal(W * H)
    return Problem("gauss2d_rot", z, truth, p0, grid=(W, H, 0), name=f"gauss2d W={W}")


def make_gauss2d_at(W: int, H: int, truth, seed: int = 30, noise: float = 0.1) -> Problem:
    """A rotated 2D Gaussian + offset with GIVEN parameters (edge cases of the
    pass: narrow, elongated, off-centre or off-image peaks); p0 = truth."""
    rng = np.random.default_rng([seed, 0])
    truth = np.asarray(truth, dtype=np.float64)
    X, Y = grid_coords(W, H)
    z = render("gauss2d_rot", (X, Y), truth) + noise * rng.standard_normal(W * H)
    return Problem("gauss2d_rot", z, truth, truth.copy(), grid=(W, H, 0), name=f"gauss2d_at W={W} H={H}")


def make_gauss2d_bounded(W: int, variant: str = "a", seed: int = 4, k: int = 0, noise: float = 0.1) -> Problem:
    """C4: as C3 with bounds.  a: loose; b: lb_off = off+0.2, ub_sx = 0.85 sx;
    c: as b with ub_sx = 0.6 sx.  p0 clipped to [lb+1e-3, ub-1e-3]."""
    pr = make_gauss2d(W, seed=seed, k=k, noise=noise)
    tr = pr.truth
    lb = np.array([0.0, 0.0, 0.0, 1.0, 1.0, -math.pi, -1.0])
    ub = np.array([10.0, W - 1.0, W - 1.0, float(W), float(W), 2 * math.pi, 2.0])
    if variant in ("b", "c"):
        lb[6] = tr[6] + 0.2
        ub[3] = (0.85 if variant == "b" else 0.6) * tr[3]
    p0 = np.clip(pr.p0, lb + 1e-3, ub - 1e-3)
    return Problem("gauss2d_rot", pr.z, tr, p0, grid=pr.grid, lb=lb, ub=ub, name=f"C4{variant} W={W}")


def make_gauss2d_x2(W: int, seed: int = 5, k: int = 0, noise: float = 0.1, H: int | None = None) -> Problem:
    """C5: two rotated 2D Gaussians + shared offset, p0 = truth (1 +- 10%)."""
    H = W if H is None else H
    rng = np.random.default_rng([seed, k])
    truth, p0 = _draw(rng, _ranges_gauss2d_x2(W), "gauss2d_rot_x2", 0.1)
    X, Y = grid_coords(W, H)
    z = render("gauss2d_rot_x2", (X, Y), truth) + noise * rng.standard_normal(W * H)
    return Problem("gauss2d_rot_x2", z, truth, p0, grid=(W, H, 0), name=f"gauss2d_x2 W={W}")


def make_linear(m: int = 200, seed: int = 11, k: int = 0, noise: float = 0.3) -> Problem:
    """Linear model x0*t + x1 (closed-form pin)."""
    rng = np.random.default_rng([seed, k])
    truth = np.array([rng.uniform(-3, 3), rng.uniform(-3, 3)])
    t = np.linspace(-1.0, 2.0, m)
    z = render("linear", t, truth) + noise * rng.standard_normal(m)
    return Problem("linear", z, truth, np.array([0.5, -0.5]), t=t, name=f"linear m={m}")


def shard_rows(H: int, R: int, k: int) -> tuple[int, int]:
    """Row band [r0, r1) of rank k out of R: floor(kH/R)."""
    return (k * H) // R, ((k + 1) * H) // R


def shard_range(m: int, R: int, k: int) -> tuple[int, int]:
    """Index range of rank k out of R for 1-D data."""
    return (k * m) // R, ((k + 1) * m) // R


C2_SWEEP = [int(v) for v in np.unique(np.round(np.logspace(3, 7, 15)).astype(np.int64))]

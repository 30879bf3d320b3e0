"""Development probe: the n = 13 moment J-pass on tiny / odd image shapes against the oracle."""
import math
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import datagen as dg  # noqa: E402
import paper_2208_12187_b200 as jf  # noqa: E402
from oracle import passes as orp  # noqa: E402

for H in (1, 3, 17):
    for W in (1, 2, 31, 33, 257, 511, 1000):
        truth = np.array([1.3, 0.37 * W, 0.61 * H, 80.0, 55.0, 0.4, 0.9, 0.55 * W, 0.3 * H, 60.0, 90.0, 1.1, 0.25])
        X, Y = dg.grid_coords(W, H)
        z = dg.render("gauss2d_rot_x2", (X, Y), truth) + 0.1 * np.random.default_rng(3).standard_normal(W * H)
        cr, gr, Gr, br = orp.jpass("gauss2d_rot_x2", (X, Y), z, truth)
        c, g, G, b = jf.jpass("gauss2d_rot_x2", z, truth, grid=(W, H, 0))
        d = np.sqrt(np.diag(Gr))
        e = max(abs(c - cr) / cr, np.max(np.abs(g - gr) / (d * math.sqrt(2 * cr))), np.max(np.abs(G - Gr) / np.outer(d, d)))
        print(f"W={W:5d} H={H:3d} max rel {e:.1e} {'FAIL' if e > 1e-10 else ''}")

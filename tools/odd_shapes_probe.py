import sys, math; sys.path.insert(0, ".")
import numpy as np, torch
import datagen as dg, paper_2208_12187_b200 as jf
from oracle import passes as orp
for H in (1, 3, 17):
    for W in (1, 2, 31, 33, 511, 512, 513, 1000, 2049):
        truth = np.array([1.3, 0.37 * W, 0.61 * H, 80.0, 55.0, 0.4, 0.25])
        pr = dg.make_gauss2d_at(W, H, truth)
        cr, gr, Gr, br = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
        c, g, G, b = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
        d = np.sqrt(np.diag(Gr))
        ec = abs(c - cr) / cr
        eg = np.max(np.abs(g - gr) / (d * math.sqrt(2 * cr)))
        eG = np.max(np.abs(G - Gr) / np.outer(d, d))
        flag = "FAIL" if max(ec, eg, eG) > 1e-10 else ""
        print(f"W={W:5d} H={H:3d} cost {ec:.1e} g {eg:.1e} G {eG:.1e} {flag}")

import sys, math; sys.path.insert(0, ".")
import numpy as np
import datagen as dg, paper_2208_12187_b200 as jf
from oracle import passes as orp
np.set_printoptions(precision=6, linewidth=200)
for (W, H) in ((1, 1), (2, 3)):
    truth = np.array([1.3, 0.37 * W, 0.61 * H, 80.0, 55.0, 0.4, 0.25])
    pr = dg.make_gauss2d_at(W, H, truth)
    cr, gr, Gr, br = orp.jpass(pr.model, pr.coords(), pr.z, pr.p0)
    c, g, G, b = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    d = np.sqrt(np.diag(Gr))
    print(W, H, "rel err matrix:\n", np.abs(G - Gr) / np.outer(d, d))
    print("Gr diag", np.diag(Gr))
    c2, g2, G2, b2 = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid, alt_coords=True)
    print("alt diag", np.diag(G2))

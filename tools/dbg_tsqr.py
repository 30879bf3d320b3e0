import os, sys, numpy as np
sys.path.insert(0, ".")
import datagen as dg
import paper_2208_12187_b200 as jf
from oracle import trf as otrf
pr = dg.make_gauss2d_bounded(256, "c")
ref = otrf.fit(pr.model, pr.coords(), pr.z, pr.p0, pr.lb, pr.ub)
print("oracle", ref["status"], ref["nfev"], ref["njev"], ref["nit"])
for graph in (True, False):
    for pol in ("speculative", "conservative"):
        r = jf.curve_fit(pr.model, pr.z, p0=pr.p0, lb=pr.lb, ub=pr.ub, grid=pr.grid, solver="tsqr", policy=pol, use_graph=graph)
        print(os.environ.get("JF_JVARIANT", "-"), "graph" if graph else "host", pol, r.status, r.nfev, r.njev, r.nit, np.max(np.abs(r.x - ref["x"]) / np.abs(ref["x"])))

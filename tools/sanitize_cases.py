"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of libjfb200.so on sizes that span several
tiles and a ragged tail.  Run by tools/sanitize.sh on the GPU box.
    python tools/sanitize_cases.py [graph]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen as dg  # noqa: E402
import paper_2208_12187_b200 as jf  # noqa: E402

use_graph = len(sys.argv) > 1 and sys.argv[1] == "graph"
torch.cuda.set_device(0)
# moment J-pass (n = 7, TMA ring), residual pass, device-x pass without the precomputed prologue
pr = dg.make_gauss2d(300, H=97, seed=3)
print("gauss2d jpass", jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)[0])
print("gauss2d rpass", jf.residual_pass(pr.model, pr.z, pr.p0, grid=pr.grid)[0])
zd = torch.as_tensor(pr.z).cuda()
kv = torch.zeros(64, dtype=torch.float64, device="cuda")
jf.pass_device(pr.model, zd, torch.as_tensor(pr.p0).cuda(), kv, grid=pr.grid)
torch.cuda.synchronize()
# odd width (no bulk copies: lanes stage the chunks), narrow peak (dual-number fallback)
po = dg.make_gauss2d(301, H=33, seed=4)
print("gauss2d odd W", jf.jpass(po.model, po.z, po.p0, grid=po.grid)[0])
xn = po.p0.copy()
xn[3] = xn[4] = 3.0
print("gauss2d narrow", jf.jpass(po.model, po.z, xn, grid=po.grid)[0])
# two-Gaussian moment kernel, weighted dual kernel, explicit coordinates
p2 = dg.make_gauss2d_x2(256, H=64, seed=5)
print("gauss2d_x2 jpass", jf.jpass(p2.model, p2.z, p2.p0, grid=p2.grid)[0])
sig = np.full(pr.m, 0.1)
print("weighted", jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid, sigma=sig)[0])
for mk in (dg.make_exp_decay, dg.make_gauss1d):
    p1 = mk(m=3001)
    print(p1.model, jf.jpass(p1.model, p1.z, p1.p0, y=p1.t)[0])
# fits: single-block small fit, fused moment fit (host loop or graph), Gram / TSQR, bounded, conservative
p1 = dg.make_exp_decay(m=1000)
print("small fit", jf.curve_fit(p1.model, p1.z, y=p1.t, p0=p1.p0).status)
pf = dg.make_gauss2d(256, seed=3)
for solver in ("auto", "tsqr"):
    r = jf.curve_fit(pf.model, pf.z, p0=pf.p0, grid=pf.grid, use_graph=use_graph, solver=solver)
    print("fit", solver, r.status, r.nfev)
r = jf.curve_fit(pf.model, pf.z, p0=pf.p0, grid=pf.grid, use_graph=use_graph, policy="conservative")
print("fit conservative", r.status, r.nfev)
lb = np.full(7, -np.inf)
ub = np.full(7, np.inf)
lb[3] = pf.p0[3] * 0.95
r = jf.curve_fit(pf.model, pf.z, p0=pf.p0, grid=pf.grid, lb=lb, ub=ub, use_graph=use_graph)
print("fit bounded", r.status, r.nfev)
# batched small fits
pb = [dg.make_exp_decay(m=200, k=k) for k in range(8)]
zb = np.stack([p.z for p in pb])
rb = jf.curve_fit_batch("exp_decay", zb, y=pb[0].t, shared_y=True, p0=np.ones((8, 3)))
print("batch", rb.status.tolist())

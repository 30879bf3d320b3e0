import sys; sys.path.insert(0, ".")
import numpy as np, torch
import datagen as dg, paper_2208_12187_b200 as jf
pr = dg.make_gauss2d(4096, seed=6)
z = torch.as_tensor(pr.z).cuda()
for i in range(4):
    r = jf.curve_fit(pr.model, z, p0=pr.p0, grid=pr.grid)
print("status", r.status, r.nfev)
print("epilogue cycles per fit [load, gn(general), prologue, step total(fast+general), after_trial, accept, outer_top, trial_finish]:", [int(c) for c in r.epilogue_cycles])
tl = np.array(r.timeline_ns) / 1e3
print("timeline", " ".join(f"{v:.1f}" for v in tl))

"""Development aid (JF_DEV build): per-step phases of the fused solver step of
a T fit from the fit's profiling counters.
    JF_DEV=1 python -m paper_2208_12187_b200.build --force; python tools/dev_solver_prof.py"""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import datagen as dg  # noqa: E402
import paper_2208_12187_b200 as jf  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
pr = dg.make_gauss2d(W, seed=6 if W == 4096 else 3)
z = torch.as_tensor(pr.z).cuda()
for i in range(4):
    r = jf.curve_fit(pr.model, z, p0=pr.p0, grid=pr.grid)
c = np.array(r.epilogue_cycles) / r.nfev / 1965.0
print(f"W={W} status {r.status} nfev {r.nfev}; us per step: load {c[0]:.2f}, prologue {c[2]:.2f}, "
      f"step (fast or general) {c[3]:.2f}, write-back {c[5]:.2f} (accept counter shares the slot); "
      f"fast path (x nfev/4): decide {c[1]:.2f} bhat+chol {c[4]:.2f} solves {c[6]:.2f} pred+commit {c[7]:.2f}")
tl = np.array(r.timeline_ns) / 1e3
print("timeline", " ".join(f"{v:.1f}" for v in tl))

"""Per-pass timing for a model/size (development aid): python tools/quick_time2.py MODEL W"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import datagen as dg
import paper_2208_12187_b200 as jf

model = sys.argv[1]
W = int(sys.argv[2])
make = {"gauss2d_rot": lambda: dg.make_gauss2d(W, seed=6), "gauss2d_rot_x2": lambda: dg.make_gauss2d_x2(W, seed=5),
        "gauss1d": lambda: dg.make_gauss1d(W), "exp_decay": lambda: dg.make_exp_decay(m=W)}[model]
pr = make()
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
z = torch.as_tensor(pr.z).cuda()
x = torch.as_tensor(pr.p0).cuda()
kv = torch.zeros(128, dtype=torch.float64, device="cuda")
kw = dict(grid=pr.grid) if pr.grid is not None else (dict(t0=pr.meta["t0"], dt=pr.meta["dt"]) if "t0" in pr.meta else dict(y=torch.as_tensor(pr.t).cuda()))
for ro in (False, True):
    for _ in range(3):
        jf.pass_device(pr.model, z, x, kv, stream=s.cuda_stream, residual_only=ro, **kw)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    N = 20
    e0.record()
    for _ in range(N):
        jf.pass_device(pr.model, z, x, kv, stream=s.cuda_stream, residual_only=ro, **kw)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / N
    print(f"{model} {'r' if ro else 'J'}-pass m={pr.m}: {t*1e3:.1f} us  {pr.m/t*1e3:.3e} pts/s")
zz = torch.as_tensor(pr.z).cuda() if pr.grid is not None else torch.as_tensor(pr.z).cuda()
fk = dict(kw)
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = jf.curve_fit(pr.model, zz, p0=pr.p0, stream=s.cuda_stream, **fk)
    torch.cuda.synchronize(); t1 = time.perf_counter()
print("fit", r.status, r.nfev, r.njev, f"{(t1-t0)*1e3:.3f} ms", "epi", f"{r.t_epilogue_s*1e6:.1f} us",
      "t_solve", f"{r.t_solve_s*1e6:.1f} us", "t_upload", f"{r.t_upload_s*1e6:.1f} us")
print("timeline us:", " ".join(f"{v/1e3:.1f}" for v in r.timeline_ns))

"""Quick per-pass timing on the GPU (development aid; bench.py is the contract)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import datagen as dg
import paper_2208_12187_b200 as jf

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
pr = dg.make_gauss2d(W, seed=6)
z = torch.as_tensor(pr.z).cuda()
x = torch.as_tensor(pr.p0).cuda()
kv = torch.zeros(64, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for ro in (False, True):
    for _ in range(3):
        jf.pass_device(pr.model, z, x, kv, grid=pr.grid, stream=s.cuda_stream, residual_only=ro, x_host=pr.p0)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    N = 50
    e0.record()
    for _ in range(N):
        jf.pass_device(pr.model, z, x, kv, grid=pr.grid, stream=s.cuda_stream, residual_only=ro, x_host=pr.p0)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / N
    print(f"{'r' if ro else 'J'}-pass W={W}: {t*1e3:.1f} us  {pr.m/t*1e3:.3e} pts/s")
    try:  # the same launches captured in a CUDA graph: kernel time without the host calls
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(N):
                jf.pass_device(pr.model, z, x, kv, grid=pr.grid, stream=s.cuda_stream, residual_only=ro, x_host=pr.p0)
        g.replay(); torch.cuda.synchronize()
        e0.record(s); g.replay(); e1.record(s); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / N
        print(f"{'r' if ro else 'J'}-pass W={W} (graph): {t*1e3:.1f} us  {pr.m/t*1e3:.3e} pts/s")
    except Exception as ex:
        print("graph timing failed:", ex)
if len(sys.argv) > 2 and sys.argv[2] == "passonly":
    sys.exit(0)
for mode in ("graph", "hostloop"):
    for i in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = jf.curve_fit(pr.model, z, p0=pr.p0, grid=pr.grid, use_graph=(mode == "graph"), stream=s.cuda_stream)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    tl = np.array(r.timeline_ns) / 1e3
    print("timeline us:", " ".join(f"{v:.1f}" for v in tl))
    print(mode, "fit", r.status, r.nfev, r.njev, r.cost, f"{(t1-t0)*1e3:.3f} ms", r.kernel_launches, f"epi {r.t_epilogue_s*1e6:.1f} us", [int(c) for c in r.epilogue_cycles])

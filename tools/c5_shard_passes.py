"""One rank's share of the C5 J-pass (8192 x 8192/N rows, n = 13) timed on one
GPU for N = 1, 2, 4, 8 (20 launches in a CUDA graph, prologue precomputed as
in a fit) — the per-rank work of the strong-scaling configuration, without
the cross-rank combine (development aid; no scaling claim)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import datagen as dg  # noqa: E402
import paper_2208_12187_b200 as jf  # noqa: E402

pr = dg.make_gauss2d_x2(8192, seed=5)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
rows = []
for N in (1, 2, 4, 8):
    r0, r1 = dg.shard_rows(8192, N, 0)
    z = torch.as_tensor(pr.z[r0 * 8192:r1 * 8192]).cuda()
    x = torch.as_tensor(pr.p0).cuda()
    kv = torch.zeros(160, dtype=torch.float64, device="cuda")
    kw = dict(grid=(8192, r1 - r0, r0), stream=s.cuda_stream, x_host=pr.p0)
    for _ in range(3):
        jf.pass_device(pr.model, z, x, kv, **kw)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            jf.pass_device(pr.model, z, x, kv, **kw)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    rows.append({"N": N, "rows_per_rank": r1 - r0, "m_per_rank": z.numel(), "jpass_us": us,
                 "ideal_us_from_N1": None})
    del z
for r in rows:
    r["ideal_us_from_N1"] = rows[0]["jpass_us"] / r["N"]
    print(json.dumps(r))

"""Where a fit's time goes outside the device work (development aid):
Python binding, C entry (staging, graph launch, copies, sync), device timeline.
    python tools/host_overhead.py [W]"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen as dg  # noqa: E402
import paper_2208_12187_b200 as jf  # noqa: E402
from paper_2208_12187_b200 import _lib as L  # noqa: E402
from paper_2208_12187_b200 import api  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
pr = dg.make_gauss2d(W, seed=6 if W == 4096 else 3)
z = torch.as_tensor(pr.z).cuda()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for _ in range(3):
    r = jf.curve_fit(pr.model, z, p0=pr.p0, grid=pr.grid, stream=s.cuda_stream)
N = 20
t0 = time.perf_counter()
for _ in range(N):
    r = jf.curve_fit(pr.model, z, p0=pr.p0, grid=pr.grid, stream=s.cuda_stream)
t_py = (time.perf_counter() - t0) / N
# the C entry alone, arguments prebuilt
lib = L.load()
mid = api._model_id(pr.model)
opts, keep = api.make_opts(grid=pr.grid, on_device=True, stream=s.cuda_stream)
res = L.jf_result()
p0 = np.ascontiguousarray(pr.p0, dtype=np.float64)
t0 = time.perf_counter()
for _ in range(N):
    lib.jf_curve_fit(mid, None, z.data_ptr(), pr.m, p0.ctypes.data, 7, None, None, C.byref(opts), C.byref(res))
t_c = (time.perf_counter() - t0) / N
# CUDA events around the call (the bench's measure)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(N):
    e0.record(s)
    r = jf.curve_fit(pr.model, z, p0=pr.p0, grid=pr.grid, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
tl = np.array(r.timeline_ns) / 1e3
print(f"W={W} nfev={r.nfev}: python {t_py*1e6:.1f} us, C call {t_c*1e6:.1f} us, events {np.median(ts)*1e3:.1f} us, "
      f"device span {tl[-1]:.1f} us, t_solve_s {r.t_solve_s*1e6:.1f} us")
print("timeline:", " ".join(f"{v:.1f}" for v in tl))

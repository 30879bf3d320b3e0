"""Per-warp timeline of one moment_stream_kernel pass (development aid).
JF_DEBUG_STAMPS=/path python tools/quick_time.py 4096 passonly; python tools/stamps2.py /path
Per warp (globaltimer ns): [smid, entry, prologue done, loop done, block partial stored]; last-block
tail (clock64, from the grid_reduce1 ticket [1]): [10] partial loads, [2] reduced, [3] returned,
[5] moments->kvec, [6] chain, [7] hand-off."""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64)
tail = raw[-16:].astype(np.int64)
d = raw[: 8000 * 8].reshape(-1, 8).astype(np.int64)
d = d[d[:, 1] > 0]
t0 = d[:, 1].min()
rel = lambda c: (d[:, c] - t0) / 1e3
en, pro, lo, pa = rel(1), rel(2), rel(3), rel(4)
q = lambda v: f"min {v.min():.2f} med {np.median(v):.2f} p90 {np.percentile(v, 90):.2f} max {v.max():.2f}"
print(f"warps {len(d)}")
print("entry      ", q(en))
print("prologue   ", q(pro), " (dur", q(pro - en), ")")
print("loop end   ", q(lo), " (dur", q(lo - pro), ")")
print("tail end   ", q(pa), " (tail dur", q(pa - lo), ")")
tl = np.where(tail > 0, tail - tail[1], 0) / 1.9e3
print("tail us from ticket [1]:", " ".join(f"[{i}] {tl[i]:.2f}" for i in (2, 5, 6, 7)))
sm = d[:, 0]
us = np.unique(sm)
first = np.array([lo[sm == s].min() for s in us])
last = np.array([lo[sm == s].max() for s in us])
print("per-SM first loop end", q(first))
print("per-SM last loop end ", q(last))
print("per-SM spread (last-first)", q(last - first))

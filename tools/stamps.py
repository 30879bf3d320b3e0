"""Per-warp timeline of one moment-kernel pass (development aid).
JF_DEBUG_STAMPS=/path python tools/quick_time.py 4096 passonly; python tools/stamps.py /path"""
import sys
import numpy as np

d = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 4)
t_end = int(d[-1, 3])
tail = d.reshape(-1)[-16:].astype(np.int64)
d = d[:16384 - 8]
d = d[d[:, 1] > 0].astype(np.int64)
t0 = d[:, 1].min()
sm, st, lo, ex = d[:, 0], (d[:, 1] - t0) / 1e3, (d[:, 2] - t0) / 1e3, (d[:, 3] - t0) / 1e3
print(f"warps {len(d)}  start: min 0 med {np.median(st):.2f} max {st.max():.2f} us")
print(f"loop end: min {lo.min():.2f} med {np.median(lo):.2f} p90 {np.percentile(lo, 90):.2f} max {lo.max():.2f} us")
print(f"loop duration: min {(lo - st).min():.2f} med {np.median(lo - st):.2f} max {(lo - st).max():.2f} us")
print(f"block partial done: med {np.median(ex):.2f} max {ex.max():.2f} us")
smend = np.array([lo[sm == s].max() for s in np.unique(sm)])
smdur = np.array([(lo[sm == s] - st[sm == s]).mean() for s in np.unique(sm)])
print(f"per-SM last loop end: min {smend.min():.2f} med {np.median(smend):.2f} max {smend.max():.2f}; "
      f"per-SM mean loop duration: min {smdur.min():.2f} med {np.median(smdur):.2f} max {smdur.max():.2f}")
order = np.argsort(smdur)
print("slowest SMs:", [(int(s), round(float(x), 2)) for s, x in zip(np.unique(sm)[order[-6:]], smdur[order[-6:]])])
print("fastest SMs:", [(int(s), round(float(x), 2)) for s, x in zip(np.unique(sm)[order[:6]], smdur[order[:6]])])
tail = np.where(tail > 0, tail - tail[1], np.nan) / 1.9e3  # clock64 -> us at ~1.9 GHz, from [1]
print("last block tail (us): [1] L1 ticket, [2] reduced, [3] finish start, [8] kvec (1st), [9] chain (1st), "
      "[4] prologue, [5] kvec, [6] chain, [7] hand-off:")
print("   ", " ".join(f"[{i}] {tail[i]:.2f}" for i in (1, 10, 2, 3, 8, 9, 4, 5, 6, 7) if not np.isnan(tail[i])),
      f"(loop end max {lo.max():.2f}, block partial max {ex.max():.2f})")

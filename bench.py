#!/usr/bin/env python
"""bench.py — the B200 hot path of JAXFit's TRF solver (arXiv 2208.12187) on
its north-star workload, printing ONE JSON line (driver contract).

Workload at N = 1 (SURVEY §8(d) "T", BASELINE.json north star): 2D rotated
Gaussian + offset, n = 7, 4096 x 4096 implicit pixel grid (m = 16,777,216),
datagen seed 6.  A STEP is one complete fit (every §8(a) row: the J-passes
with fused Gram reduction, the device subproblem, the control, the graph
driver) on data already resident in HBM.  With N > 1 ranks (torchrun) the
workload is BASELINE config 5 (C5): two rotated Gaussians, n = 13, one
8192 x 8192 image split into N row bands of 8192/N rows (strong scaling),
fitted as ONE problem: each pass combines the ranks' K-vectors inside the
pass kernel over NVLink (jf_comm mailboxes).  At N = 1 the same C5 fit is
reported as a secondary result ("c5") so the scaling curve has its N = 1
point; "batch" reports the batched many-small-fits path (N2).

    value = points processed per second per pass = m_total * passes / t_fit
    (passes per fit = the J-passes the speculative policy runs = nfev)

Also reported: the dominant kernel (J-pass) against the FP64 roofline
(DESIGN.md §6), the oracle as CPU baseline, an end-to-end number through the
public API from host memory, clocks during the timed region.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen as dg  # noqa: E402

W_IMG = 4096
SEED = 6
N_PARAMS = 7
# Roofline of the n=7 J-pass: per point it must read z (8 B,
# implicit grid) and, in the moment form (jf_moment.cuh), execute 19 fp64
# operations (row recurrence 2, residual 2, u^2 1, u r 1, the eleven
# step-index moments 11, sum r and sum r^2 2; per-chunk/per-task overheads
# are the implementation's, not the algorithm's).  HBM: 8 B per
# point at the measured HBM peak; FP64: 19 / (148 SMs x 64 lanes x 1.965 GHz)
# per point -> at 4096^2 20.5 us vs 17.1 us: the pass is HBM-bound and is reported against the
# measured HBM peak (MEASURED_PEAKS.json hbm_gbs), with the FP64-pipe
# fraction alongside.  (The dual-number rank-1 form needs 85 fp64 per point,
# SURVEY §8(d) d.3, and would be FP64-bound.)
ALG_FP64_INSTR_PER_POINT = 19
BYTES_PER_POINT = 8  # z only (implicit grid)
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: SMs x FP64 lanes x 2 x max SM clock
J_KERNEL = "moment_stream_kernel<16, 12, 8, 3>"


def fp64_peak():
    """Measured DFMA throughput (tools/fp64_peak.cu -> profiles/fp64_peak.json), else nominal."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        return float(d["dfma_tflops"]), "profiles/fp64_peak.json dfma_tflops (measured DFMA, tools/fp64_peak.cu)"
    except Exception:
        return FP64_NOMINAL_TFLOPS, "nominal 148 SMs x 64 FP64 lanes x 2 x 1.965 GHz"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev):
        self.dev = dev
        self.p = None
        self.path = os.path.join("/tmp", f"jf_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.15)
            self.p.terminate()
            try:
                self.p.wait(timeout=2)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 3 + k and "Active" in r[3 + k] and "Not" not in r[3 + k]:
                    reasons.add(nm)
        load = [v for v in sm if v > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def _oracle_band_worker(args):
    """One host process: the oracle's J-pass over a band of the image, repeated
    for budget_s seconds; returns the points processed and the seconds."""
    model, W, r0, rows, z, x, budget_s = args
    from oracle import passes as orp
    X, Y = dg.grid_coords(W, rows, r0)
    t0 = time.perf_counter()
    reps = 0
    while True:
        orp.jpass(model, (X, Y), z, x)
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return reps * rows * W, time.perf_counter() - t0


def cpu_baseline_oracle(pr, budget_s=8.0, rows=64):
    """The oracle's J-pass (oracle/passes.py, as it stands) on a bounded sample
    of the same workload, timed on one host core and on all of them (one
    process per core, each on its own band of rows; points/s summed)."""
    import multiprocessing as mp
    W, H = pr.grid[0], pr.grid[1]
    ncore = os.cpu_count() or 1
    bands = []
    for k in range(ncore):
        r0 = (k * rows) % max(1, H - rows)
        bands.append((pr.model, W, r0, rows, pr.z[r0 * W:(r0 + rows) * W], pr.p0, budget_s))
    pts1, dt1 = _oracle_band_worker(bands[0])
    os.environ["OMP_NUM_THREADS"] = "1"
    with mp.get_context("fork").Pool(ncore) as pool:  # (the workers touch no CUDA state)
        res = pool.map(_oracle_band_worker, bands)
    allc = sum(p for p, _ in res) / max(t for _, t in res)
    return {"value": allc, "unit": "points/s", "cores": ncore, "kind": "oracle",
            "sample": f"oracle J-pass (oracle/passes.py) over {rows}-row bands of the {W}x{W} image, "
                      f"{ncore} processes x ~{budget_s:.0f} s", "value_1core": pts1 / dt1, "cores_1core": 1}


def run_reference(args):
    """--impl reference: the oracle TRF (oracle/trf.py, as it stands) on the
    host cores, each step a bounded sample of the workload (a 256-row band of
    the 4096^2 image fitted as its own problem)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import trf as otrf
    if world == 1:  # T: a 256-row band of the 4096^2 image
        pr = dg.make_gauss2d(W_IMG, seed=SEED)
        W, rows = W_IMG, 256
        metric = "data points/s per J-pass (complete TRF fits, 2D Gaussian n=7)"
        desc, scaling = f"gauss2d_rot n=7, rows 0..{rows} of the {W}x{W} seed-{SEED} image (bounded sample of T)", "weak"
    else:  # N > 1: our arm's C5 metric; a 64-row band of the 8192^2 two-Gaussian image (n = 13)
        W, rows = 8192, 64
        pr = dg.make_gauss2d_x2(W, seed=5, H=rows)
        metric = "data points/s per J-pass (complete TRF fits, two 2D Gaussians n=13, C5 row bands)"
        desc, scaling = f"gauss2d_rot_x2 n=13, rows 0..{rows} of the {W}x{W} seed-5 image (bounded sample of C5)", "strong"
    z = pr.z[: rows * W]
    X, Y = dg.grid_coords(W, rows, 0)
    times, pts = [], []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = otrf.fit(pr.model, (X, Y), z, pr.p0)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            pts.append(z.size * r["nfev"])
    tot = sum(times)
    value = sum(pts) / tot
    line = {
        "impl": "reference", "metric": metric,
        "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "m": int(z.size), "parallelism": "oracle on rank 0's host cores"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle/trf.py fit of a {rows}x{W} band per step"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_fits(jf, torch, model, z_dev, kw, steps, warmup, flush, stream, barrier, clk=None):
    """warmup untimed fits, then `steps` fits each bracketed by CUDA events on
    the fit's stream, L2 flushed before each (outside the events)."""
    res = None
    for _ in range(warmup):
        res = jf.curve_fit(model, z_dev, **kw)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    passes = launches = 0
    ctx = clk if clk is not None else _Null()
    with ctx:
        for k in range(steps):
            flush.zero_()
            ev[k][0].record(stream)
            res = jf.curve_fit(model, z_dev, **kw)
            ev[k][1].record(stream)
            passes += res.nfev
            launches += res.kernel_launches
        barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    return t_ms, passes, launches, res


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def time_jpass(jf, torch, model, z_dev, x_dev, grid, stream, comm=None, m_global=0, NJ=20, x_host=None):
    """Average J-pass launch duration: NJ back-to-back launches captured in a
    CUDA graph (a bare kernel launch each), CUDA events on the launch stream.
    x_host: the host copy of x (the pass's parameter-only prologue is then
    precomputed by the call, as the solver kernel does inside a fit)."""
    kv = torch.zeros(160, dtype=torch.float64, device="cuda")
    pkw = dict(grid=grid, stream=stream.cuda_stream, x_host=x_host)
    if comm is not None:
        pkw.update(comm=comm, m_global=m_global)
    for _ in range(3):
        jf.pass_device(model, z_dev, x_dev, kv, **pkw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = None
    if comm is None:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(NJ):
                    jf.pass_device(model, z_dev, x_dev, kv, **pkw)
            g.replay()
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001
            print(f"# J-pass graph capture failed ({ex}); timing host-issued launches", file=sys.stderr)
            g = None
            torch.cuda.synchronize()
    e0.record(stream)
    if g is not None:
        g.replay()
    else:
        for _ in range(NJ):
            jf.pass_device(model, z_dev, x_dev, kv, **pkw)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / NJ * 1e-3


def batch_measure(jf, torch, nfits=20000, m=1000, reps=5):
    """N2: nfits independent C1-sized fits (exp decay, m = 1000, SURVEY d.2 C1
    recipe per fit index k) in ONE launch; fits/s with the data resident, and
    end to end from pinned host memory; the oracle's fits/s on one host core."""
    from oracle import trf as otrf
    probs = [dg.make_exp_decay(m=m, k=k) for k in range(64)]
    z_host = torch.empty((nfits, m), dtype=torch.float64, pin_memory=True)
    zn = z_host.numpy()
    for k in range(nfits):
        zn[k] = probs[k % 64].z
    t = probs[0].t
    z_dev = z_host.cuda()
    t_dev = torch.as_tensor(t).cuda()
    p0 = np.ones((nfits, 3))
    kw = dict(y=t_dev, shared_y=True, p0=p0)
    for _ in range(2):
        r = jf.curve_fit_batch("exp_decay", z_dev, **kw)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        r = jf.curve_fit_batch("exp_decay", z_dev, **kw)
    e1.record(s)
    torch.cuda.synchronize()
    t_dev_s = e0.elapsed_time(e1) * 1e-3 / reps
    re = jf.curve_fit_batch("exp_decay", z_host.numpy(), y=t, shared_y=True, p0=p0)  # (staging buffers sized)
    t0 = time.perf_counter()
    for _ in range(reps):
        re = jf.curve_fit_batch("exp_decay", z_host.numpy(), y=t, shared_y=True, p0=p0)
    t_e2e = (time.perf_counter() - t0) / reps
    # oracle on one host core, bounded sample (the same fits)
    c0 = time.perf_counter()
    nor = 0
    while time.perf_counter() - c0 < 4.0:
        otrf.fit("exp_decay", t, probs[nor % 64].z, np.ones(3))
        nor += 1
    t_or = (time.perf_counter() - c0) / nor
    ok = int(np.sum(r.status > 0))
    return {"workload": f"C1 exp_decay a*exp(-b t)+c, m={m}, {nfits} independent fits per launch (one warp per fit)",
            "value": nfits / t_dev_s, "unit": "fits/s", "ms_per_launch": t_dev_s * 1e3, "fits_converged": ok,
            "mean_nfev": float(np.mean(r.nfev)),
            "e2e": {"value": nfits / t_e2e, "unit": "fits/s", "h2d_bytes_per_step": int(z_host.numel() * 8 + t.nbytes + p0.nbytes),
                    "d2h_bytes_per_step": int(nfits * (16 * 8 + 16 + 16))},
            "cpu_baseline": {"value": 1.0 / t_or, "unit": "fits/s", "cores": 1, "kind": "oracle",
                             "sample": f"oracle/trf.py fits of the same C1 problems, {nor} fits"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="host-driven loop instead of the CUDA graph (ncu cannot see kernels inside conditional graph nodes)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import paper_2208_12187_b200 as jf

    rank, world, local = dist_env()
    local = local % torch.cuda.device_count()  # (a 1-GPU smoke test of the N > 1 path puts every rank on cuda:0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        backend = os.environ.get("JF_BENCH_BACKEND", "nccl")  # gloo: ranks sharing one GPU (smoke test only)
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
        dist = tdist
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist is None or dist.get_backend() == "nccl" else "cpu")
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peak64, peak64_src = fp64_peak()
    hbm_peak = 6467.1
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass

    if world == 1:
        model = "gauss2d_rot"
        W, H = W_IMG, W_IMG
        pr = dg.make_gauss2d(W_IMG, seed=SEED)
        r0, r1 = 0, H
        scaling = "weak"
        wl = f"T: gauss2d_rot n=7, {W}x{H} implicit grid, seed {SEED}"
    else:  # C5 strong scaling: one 8192^2 image, row bands
        model = "gauss2d_rot_x2"
        W = H = 8192
        pr = dg.make_gauss2d_x2(W, seed=5)
        r0, r1 = dg.shard_rows(H, world, rank)
        scaling = "strong"
        wl = f"C5: gauss2d_rot_x2 n=13, {W}x{H} implicit grid, seed 5, {world} row bands of ~{H // world} rows"
    z_pin = torch.empty(((r1 - r0) * W,), dtype=torch.float64, pin_memory=True)  # e2e: pinned host input
    z_pin.numpy()[:] = pr.z[r0 * W: r1 * W]
    z_host = z_pin.numpy()
    m_local, m_total = z_host.size, pr.m
    grid = (W, r1 - r0, r0)
    z_dev = torch.as_tensor(z_host).cuda()
    comm = jf.Comm.from_process_group(rank, world, local, dist) if world > 1 else None
    kw = dict(grid=grid, p0=pr.p0, stream=stream.cuda_stream, use_graph=not args.no_graph)
    if comm is not None:
        kw.update(comm=comm, m_global=m_total)

    # ---- headline: K complete fits (warmup includes the one-time graph instantiation)
    clk = Clocks(local)
    t_ms, passes, launches, res = time_fits(jf, torch, model, z_dev, kw, args.steps, args.warmup, flush, stream,
                                            barrier, clk)
    t_ms = max_over_ranks(t_ms)
    value = m_total * passes / (t_ms * 1e-3)

    # ---- dominant kernel: J-pass duration, CUDA events on its stream
    x_dev = torch.as_tensor(pr.p0).cuda()
    t_j = max_over_ranks(time_jpass(jf, torch, model, z_dev, x_dev, grid, stream, comm, m_total, x_host=pr.p0))
    nfp = ALG_FP64_INSTR_PER_POINT if model == "gauss2d_rot" else 41
    achieved = BYTES_PER_POINT * m_local / t_j / 1e9
    fp64_achieved = 2.0 * nfp * m_local / t_j / 1e12
    roofline = {
        "bound": "hbm", "kernel": (J_KERNEL + " (moment-form J-pass, n=7 implicit grid, fp64)") if model == "gauss2d_rot"
        else "moment2_task_kernel<8, 8, 12, true> (moment-form J-pass, n=13, fp64)",
        "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
        "traffic": None, "launch_us": t_j * 1e6,
        "alg_work": f"{BYTES_PER_POINT} B/point (z) x {m_local} points; FP64 floor {nfp} instr/point x {m_local} points",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
        "fp64_tflops": fp64_achieved, "fp64_peak_tflops": peak64, "fp64_peak_source": peak64_src,
        "fp64_frac": fp64_achieved / peak64,
        "t_floor_us": max(BYTES_PER_POINT * m_local / (hbm_peak * 1e9), nfp * m_local / (peak64 * 1e12 / 2)) * 1e6,
    }
    try:  # dram traffic of the same kernel from the committed ncu --set full capture (same kernel name only)
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic_jpass.json")))
        if model == "gauss2d_rot" and J_KERNEL.replace(" ", "") in tj.get("kernel", "").replace(" ", ""):
            roofline["traffic"] = tj["dram_bytes_per_launch"]
            roofline["traffic_source"] = tj.get("source", "profiles/traffic_jpass.json")
    except Exception:
        pass

    # ---- end to end through the public API from pinned host memory
    e2e_ms = []
    for _ in range(3):
        barrier()
        t0 = time.perf_counter()
        r = jf.curve_fit(model, z_host, **kw)
        barrier()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_passes = r.nfev
    e2e_t = max_over_ranks(statistics.median(e2e_ms))
    e2e = {"value": m_total * e2e_passes / (e2e_t * 1e-3), "unit": "points/s",
           "h2d_bytes_per_step": int(z_host.nbytes + 8 * pr.n), "d2h_bytes_per_step": int(4 * 8 * 256 + 2048),
           "fit_ms": e2e_t}

    # ---- N = 1 secondaries: the C5 point of the scaling curve, the batched small fits
    c5 = None
    if world == 1 and not args.no_c5:
        p5 = dg.make_gauss2d_x2(8192, seed=5)
        z5 = torch.as_tensor(p5.z).cuda()
        kw5 = dict(grid=p5.grid, p0=p5.p0, stream=stream.cuda_stream)
        t5, pa5, _, r5 = time_fits(jf, torch, "gauss2d_rot_x2", z5, kw5, 3, 2, flush, stream, barrier)
        tj5 = time_jpass(jf, torch, "gauss2d_rot_x2", z5, torch.as_tensor(p5.p0).cuda(), p5.grid, stream, NJ=5)
        c5 = {"workload": "C5: gauss2d_rot_x2 n=13, 8192x8192 implicit grid, seed 5 (N=1 point of the scaling curve)",
              "value": p5.m * pa5 / (t5 * 1e-3), "unit": "points/s", "fit_ms": t5 / 3, "status": r5.status,
              "nfev": r5.nfev, "njev": r5.njev, "jpass_us": tj5 * 1e6, "jpass_points_per_s": p5.m / tj5}
        del z5
    batch = None
    if world == 1 and not args.no_batch:
        batch = batch_measure(jf, torch)

    if rank == 0:
        line = {
            "metric": "data points/s per J-pass (complete TRF fits, 2D Gaussian n=7)" if world == 1 else
                      "data points/s per J-pass (complete TRF fits, two 2D Gaussians n=13, C5 row bands)",
            "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl, "m": m_total, "passes_per_fit": passes / args.steps, "nfev": res.nfev,
                       "njev": res.njev, "status": res.status, "cost": res.cost,
                       "l2": "flushed (256 MB write) between steps", "policy": "speculative", "solver": "auto",
                       "driver": "host loop" if args.no_graph else "CUDA graph, conditional WHILE node",
                       "parallelism": f"dp{world}"},
            "roofline": roofline,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "solver_epilogue_us_per_fit": res.t_epilogue_s * 1e6,
        }
        if c5 is not None:
            line["c5"] = c5
        if batch is not None:
            line["batch"] = batch
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline_oracle(pr)
        print(json.dumps(line), flush=True)
    if comm is not None:
        barrier()
        comm.destroy()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — the B200 hot path of JAXFit's TRF solver (arXiv 2208.12187) on
its north-star workload, printing ONE JSON line (driver contract).

Workload (SURVEY §8(d) "T", BASELINE.json north star): 2D rotated Gaussian +
offset, n = 7, 4096 x 4096 implicit pixel grid (m = 16,777,216), datagen seed
6.  A STEP is one complete fit (every §8(a) row: the J-passes with fused Gram
reduction, the device subproblem, the control, the graph driver) on data
already resident in HBM.  With N > 1 ranks (torchrun) the image grows with N
(4096 x 4096N, one 4096-row band per rank: weak scaling) and is fitted as ONE
problem: each pass combines the ranks' K-vectors inside the pass kernel over
NVLink (jf_comm mailboxes).

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
# are the implementation's, not the algorithm's).  HBM: 8 B / 6467 GB/s per
# point; FP64: 19 / (148 SMs x 64 lanes x 1.965 GHz) per point -> at 4096^2
# 20.8 us vs 17.1 us: the pass is HBM-bound and is reported against the
# measured HBM peak (MEASURED_PEAKS.json hbm_gbs), with the FP64-pipe
# fraction alongside.  (The dual-number rank-1 form needs 85 fp64 per point,
# SURVEY §8(d) d.3, and would be FP64-bound.)
ALG_FP64_INSTR_PER_POINT = 19
BYTES_PER_POINT = 8  # z only (implicit grid)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: SMs x FP64 lanes x 2 x max SM clock


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


def cpu_baseline_oracle(pr, budget_s=12.0):
    """The oracle's J-pass (oracle/passes.py, as it stands) on a bounded sample
    of the same workload: a band of image rows, repeated until ~budget_s."""
    from oracle import passes as orp
    W = pr.grid[0]
    rows = 256
    z = pr.z[: rows * W]
    X, Y = dg.grid_coords(W, rows, 0)
    t0 = time.perf_counter()
    reps = 0
    while True:
        orp.jpass(pr.model, (X, Y), z, pr.p0)
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": reps * rows * W / dt, "unit": "points/s", "cores": 1, "kind": "oracle",
            "sample": f"oracle J-pass over rows 0..{rows} of the {W}x{W} image ({rows * W} points) x {reps}",
            "host_cores_available": os.cpu_count()}


def run_reference(args):
    """--impl reference: the oracle TRF (oracle/trf.py, as it stands) on the
    host cores, each step a bounded sample of the workload (a 256-row band of
    the 4096^2 image fitted as its own problem)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import trf as otrf
    pr = dg.make_gauss2d(W_IMG, seed=SEED)
    rows = 256
    z = pr.z[: rows * W_IMG]
    X, Y = dg.grid_coords(W_IMG, rows, 0)
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
        "impl": "reference", "metric": "data points/s per J-pass (complete TRF fits, 2D Gaussian n=7)",
        "value": value, "unit": "points/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"gauss2d_rot n=7, rows 0..{rows} of the {W_IMG}x{W_IMG} seed-{SEED} image "
                               f"(bounded sample of T)", "m": int(z.size)},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle/trf.py fit of a {rows}x{W_IMG} band per step"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist

    # ---- data: one 4096-row band per rank of a 4096 x (4096 * world) image
    H_total = W_IMG * world
    pr_full = dg.make_gauss2d(W_IMG, seed=SEED, H=H_total) if world > 1 else dg.make_gauss2d(W_IMG, seed=SEED)
    r0, r1 = dg.shard_rows(H_total, world, rank)
    import torch as _t
    z_pin = _t.empty(((r1 - r0) * W_IMG,), dtype=_t.float64, pin_memory=True)  # e2e: pinned host input
    z_pin.numpy()[:] = pr_full.z[r0 * W_IMG: r1 * W_IMG]
    z_host = z_pin.numpy()
    m_local = z_host.size
    m_total = pr_full.m
    grid = (W_IMG, r1 - r0, r0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    z_dev = torch.as_tensor(z_host).cuda()
    comm = None
    if world > 1:
        comm = jf.Comm.from_process_group(rank, world, local, dist)
    kw = dict(grid=grid, p0=pr_full.p0, stream=stream.cuda_stream, use_graph=not args.no_graph)
    if comm is not None:
        kw.update(comm=comm, m_global=m_total)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warmup (includes the one-time graph instantiation, excluded as in P:246)
    for _ in range(args.warmup):
        res = jf.curve_fit("gauss2d_rot", z_dev, **kw)
    barrier()

    # ---- timed: K complete fits, L2 flushed between them (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    passes = 0
    launches = 0
    with Clocks(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            res = jf.curve_fit("gauss2d_rot", z_dev, **kw)
            ev[k][1].record(stream)
            passes += res.nfev
            launches += res.kernel_launches
        barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    t_max = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_ms = float(t_max.item())
    value = m_total * passes / (t_ms * 1e-3)

    # ---- dominant kernel: J-pass duration, CUDA events on its stream
    x_dev = torch.as_tensor(pr_full.p0).cuda()
    kv = torch.zeros(64, dtype=torch.float64, device="cuda")
    pkw = dict(grid=grid, stream=stream.cuda_stream)
    if comm is not None:
        pkw.update(comm=comm, m_global=m_total)
    for _ in range(3):
        jf.pass_device("gauss2d_rot", z_dev, x_dev, kv, **pkw)
    barrier()
    NJ = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # NJ back-to-back J-pass launches captured in a CUDA graph (a repeated
    # pass is a bare kernel launch: its arguments are already on the device),
    # so the events time the kernels, not the host calls that issue them
    j_graph = None
    if comm is None:
        try:
            j_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(j_graph, stream=stream):
                for _ in range(NJ):
                    jf.pass_device("gauss2d_rot", z_dev, x_dev, kv, grid=grid, stream=stream.cuda_stream)
            j_graph.replay()
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001 — fall back to host-issued launches
            print(f"# J-pass graph capture failed ({ex}); timing host-issued launches", file=sys.stderr)
            j_graph = None
            torch.cuda.synchronize()
    e0.record(stream)
    if j_graph is not None:
        j_graph.replay()
    else:
        for _ in range(NJ):
            jf.pass_device("gauss2d_rot", z_dev, x_dev, kv, **pkw)
    e1.record(stream)
    barrier()
    t_j = e0.elapsed_time(e1) / NJ * 1e-3
    hbm_peak = 6467.1
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    achieved = BYTES_PER_POINT * m_local / t_j / 1e9
    fp64_achieved = 2.0 * ALG_FP64_INSTR_PER_POINT * m_local / t_j / 1e12
    roofline = {
        "bound": "hbm", "kernel": "moment_task_kernel<16,4,12,4,0,2> (moment-form J-pass, n=7 implicit grid, fp64)",
        "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
        "traffic": None, "launch_us": t_j * 1e6,
        "alg_work": f"{BYTES_PER_POINT} B/point (z) x {m_local} points; "
                    f"FP64 floor {ALG_FP64_INSTR_PER_POINT} instr/point x {m_local} points",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
        "fp64_tflops": fp64_achieved, "fp64_peak_tflops": FP64_PEAK_TFLOPS,
        "fp64_frac": fp64_achieved / FP64_PEAK_TFLOPS,
        "t_floor_us": max(BYTES_PER_POINT * m_local / (hbm_peak * 1e9),
                          ALG_FP64_INSTR_PER_POINT * m_local / (FP64_PEAK_TFLOPS * 1e12 / 2)) * 1e6,
    }
    prof_path = os.path.join(ROOT, "profiles", "traffic_jpass.json")
    if os.path.exists(prof_path):
        try:
            roofline["traffic"] = json.load(open(prof_path)).get("dram_bytes_per_launch")
        except Exception:
            pass

    # ---- end to end through the public API from host memory
    e2e_ms = []
    for k in range(3):
        barrier()
        t0 = time.perf_counter()
        r = jf.curve_fit("gauss2d_rot", z_host, **kw)
        barrier()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_passes = r.nfev
    e2e_t = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_t = float(e2e_t.item())
    e2e = {"value": m_total * e2e_passes / (e2e_t * 1e-3), "unit": "points/s",
           "h2d_bytes_per_step": int(z_host.nbytes + 8 * N_PARAMS),
           "d2h_bytes_per_step": 2392, "fit_ms": e2e_t}

    if rank == 0:
        line = {
            "metric": "data points/s per J-pass (complete TRF fits, 2D Gaussian n=7)",
            "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"T: gauss2d_rot n=7, {W_IMG}x{H_total} implicit grid, seed {SEED}"
                                   + (f", {W_IMG}-row band per rank" if world > 1 else ""),
                       "m": m_total, "passes_per_fit": passes / args.steps, "nfev": res.nfev, "njev": res.njev,
                       "status": res.status, "cost": res.cost, "l2": "flushed (256 MB write) between steps",
                       "policy": "speculative",
                       "driver": "host loop" if args.no_graph else "CUDA graph, conditional WHILE node",
                       "parallelism": f"dp{world}"},
            "roofline": roofline,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "solver_epilogue_us_per_fit": res.t_epilogue_s * 1e6,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_oracle(pr_full)
        print(json.dumps(line), flush=True)
    if comm is not None:
        barrier()
        comm.destroy()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

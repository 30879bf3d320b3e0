"""Fit wall time and points/s per pass across the BASELINE configs (SURVEY
§8(d) d.1): C1, the C2 length sweep (the paper's fit-time-vs-length curve),
C3, C4a/b/c, T and C5 on one B200, with the oracle timed beside the small
cases on the host.  Development/measurement aid (bench.py is the contract).

    python tools/sweep.py [--out gpurun_out/sweep.json] [--fits 5]

Per config: status/nfev/njev of the fit, median device time of a complete
fit (CUDA events, data resident in HBM, graph driver), the J-pass time (20
launches captured in a CUDA graph) and points/s per J-pass, the J-pass
roofline floor max(bytes/pt / HBM, FP64 instr/pt / P64) and the fraction.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen as dg  # noqa: E402
import paper_2208_12187_b200 as jf  # noqa: E402

try:  # the measured peaks (driver-written MEASURED_PEAKS.json, profiles/fp64_peak.json)
    HBM = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
except Exception:  # noqa: BLE001
    HBM = 6467.1e9
try:
    P64 = float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dfma_tflops"]) * 1e12 / 2
except Exception:  # noqa: BLE001
    P64 = 148 * 64 * 1.965e9  # FP64 instr/s (nominal)
# FP64 instructions per point of each J-pass as built (the
# dual-number counts are SURVEY §8(d) d.3's), bytes per point of the inputs
ALG = {"exp_decay": (16, 33), "gauss1d": (8, 43), "gauss2d_rot": (8, 19), "gauss2d_rot_x2": (8, 41)}


def problems():
    yield "C1 exp_decay m=1000", dg.make_exp_decay()
    for m in dg.C2_SWEEP:
        yield f"C2 gauss1d m={m}", dg.make_gauss1d(m)
    yield "C3 gauss2d 1024^2", dg.make_gauss2d(1024, seed=3)
    for v in "abc":
        yield f"C4{v} gauss2d 1024^2 bounded", dg.make_gauss2d_bounded(1024, v)
    yield "T gauss2d 4096^2", dg.make_gauss2d(4096, seed=6)
    yield "C5 gauss2d_x2 8192^2 (1 GPU)", dg.make_gauss2d_x2(8192, seed=5)


def coord_kw(pr, dev):
    if pr.grid is not None:
        return dict(grid=pr.grid)
    if "t0" in pr.meta:
        return dict(t0=pr.meta["t0"], dt=pr.meta["dt"])
    return dict(y=torch.as_tensor(pr.t).to(dev))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--fits", type=int, default=5)
    ap.add_argument("--oracle-max-m", type=int, default=200_000)
    a = ap.parse_args()
    dev = torch.device("cuda")
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    rows = []
    for name, pr in problems():
        z = torch.as_tensor(pr.z).to(dev)
        kw = coord_kw(pr, dev)
        fk = dict(kw, p0=pr.p0, stream=s.cuda_stream)
        if pr.lb is not None:
            fk.update(lb=pr.lb, ub=pr.ub)
        for _ in range(2):
            r = jf.curve_fit(pr.model, z, **fk)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.fits):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            r = jf.curve_fit(pr.model, z, **fk)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t_fit = statistics.median(ts)
        # J-pass: 20 launches in a CUDA graph
        x = torch.as_tensor(pr.p0).to(dev)
        kv = torch.zeros(256, dtype=torch.float64, device=dev)
        pk = dict(kw, stream=s.cuda_stream, x_host=pr.p0)  # (the prologue precomputed, as in a fit)
        jf.pass_device(pr.model, z, x, kv, **pk)
        torch.cuda.synchronize()
        NJ = 20
        t_pass = None
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(NJ):
                    jf.pass_device(pr.model, z, x, kv, **pk)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            t_pass = e0.elapsed_time(e1) * 1e-3 / NJ
        except Exception as ex:  # noqa: BLE001
            print(f"# {name}: graph timing failed: {ex}", file=sys.stderr)
            torch.cuda.synchronize()
        bpp, fpp = ALG[pr.model]
        if pr.model == "exp_decay":
            bpp = 16
        floor = max(bpp * pr.m / HBM, fpp * pr.m / P64)
        row = {"config": name, "model": pr.model, "m": pr.m, "status": r.status, "nfev": r.nfev, "njev": r.njev,
               "fit_ms": t_fit * 1e3, "fit_points_per_s": pr.m * r.nfev / t_fit,
               "jpass_us": None if t_pass is None else t_pass * 1e6,
               "jpass_points_per_s": None if t_pass is None else pr.m / t_pass,
               "jpass_floor_us": floor * 1e6, "jpass_roofline_frac": None if t_pass is None else floor / t_pass,
               "floor_bound": "hbm" if bpp * pr.m / HBM >= fpp * pr.m / P64 else "fp64"}
        if pr.m <= a.oracle_max_m:
            from oracle import trf as otrf  # the oracle as it stands, host cores, beside the GPU number
            coords = pr.coords() if pr.grid is not None else pr.t
            t0 = time.perf_counter()
            ref = otrf.fit(pr.model, coords, pr.z, pr.p0, lb=pr.lb, ub=pr.ub)
            row["oracle_fit_ms"] = (time.perf_counter() - t0) * 1e3
            row["oracle_same_trajectory"] = (ref["status"], ref["nfev"], ref["njev"]) == (r.status, r.nfev, r.njev)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del z
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()

"""Summarise ncu --set full reports (development aid; run where ncu exists).

    python tools/ncu_summary.py TAG gpurun_out/jpass_TAG.ncu-rep ... > profiles/TAG_ncu_summary.txt

Also writes profiles/traffic_jpass.json from the report whose name contains
'jpass' (dram bytes per launch of the J-pass, read by bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_elapsed.avg",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__sass_inst_executed_op_local_ld.sum",
    # FP64 per-operation counts (thread instructions), FP32 pipe and SFU (the north star's ncu evidence list)
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__inst_executed_pipe_fp64.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def stalls(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    tot = {h[i][6:]: sum(int(r[i] or 0) for r in rows[2:] if len(r) == len(h)) for i in cols}
    s = sum(tot.values()) or 1
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:6]
    return ", ".join(f"{k} {100 * v / s:.0f}%" for k, v in top)


def main():
    tag = sys.argv[1]
    for path in sys.argv[2:]:
        h, units, v = raw(path)
        name = v[h.index("Kernel Name")]
        print(f"== {os.path.basename(path)}  [{tag}]")
        print(f"  Kernel Name = {name}")
        vals = {}
        for k in KEYS:
            if k in h:
                vals[k] = v[h.index(k)]
                print(f"  {k} = {vals[k]} {units[h.index(k)]}")
        try:
            print(f"  stalls: {stalls(path)}")
        except Exception as e:  # source page needs -lineinfo / --import-source
            print(f"  stalls: n/a ({e})")
        if "jpass" in os.path.basename(path):
            def b(k):
                x = float(vals[k])
                u = units[h.index(k)]
                return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            rd, wr = b("dram__bytes_read.sum"), b("dram__bytes_write.sum")
            json.dump({"kernel": name, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                       "algorithmic_bytes": 134217728, "source": f"ncu --set full, profiles/{tag}_ncu_summary.txt"},
                      open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                        "traffic_jpass.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

"""Build libjfb200.so in-tree with nvcc for sm_100a (B200).

Each csrc/*.cu is one translation unit (one per model for the pass kernels,
plus the host driver); they compile in parallel and link into a single
shared library next to this file.  Rebuilds only what changed (mtime of the
unit vs. every header and the unit itself).

    python -m paper_2208_12187_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import re
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libjfb200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
if os.environ.get("JF_DEV"):  # development build: per-warp timeline stamps, diagnostics (never shipped)
    NVCC_FLAGS += ["-DJF_DEV=1"]
if os.environ.get("JF_CHECKED"):  # checked build: device bounds checks (JF_DCHECK), never shipped
    NVCC_FLAGS += ["-DJF_CHECKED=1"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libjfb200.so")


def _deps(path: str, seen: set | None = None) -> set:
    """Files a unit includes (quoted #include, recursively): a header edit
    recompiles only the units that include it."""
    seen = set() if seen is None else seen
    with open(path) as f:
        for line in f:
            mt = re.match(r'\s*#\s*include\s+"([^"]+)"', line)
            if mt:
                dep = os.path.normpath(os.path.join(os.path.dirname(path), mt.group(1)))
                if os.path.exists(dep) and dep not in seen:
                    seen.add(dep)
                    _deps(dep, seen)
    return seen


def _stale(src: str, obj: str, hdr_mtime: float) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return t < os.path.getmtime(src) or t < hdr_mtime


def _compile(src: str, obj: str, verbose: bool) -> str:
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stderr}")
    return r.stderr


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    todo = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        hdr_mtime = max((os.path.getmtime(h) for h in _deps(s)), default=0.0)
        if force or _stale(s, o, hdr_mtime):
            todo.append((s, o))
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            futs = {ex.submit(_compile, s, o, verbose): s for s, o in todo}
            for f in cf.as_completed(futs):
                log = f.result()
                if verbose and log:
                    sys.stderr.write(f"== {os.path.basename(futs[f])}\n{log}")
    stale_lib = (not os.path.exists(LIB)) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)
    if todo or stale_lib:
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()

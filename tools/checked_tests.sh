#!/bin/bash
# The GPU suite against a checked build (device bounds checks JF_DCHECK; see
# jf_common.cuh) — the substitute for compute-sanitizer on this GPU pool.
# Run on the GPU box; the log goes to gpurun_out/checked_tests.log.
mkdir -p gpurun_out
JF_CHECKED=1 python -m paper_2208_12187_b200.build --force > gpurun_out/checked_build.log 2>&1 || { tail -20 gpurun_out/checked_build.log; exit 1; }
strings paper_2208_12187_b200/libjfb200.so | grep -c "JF_DCHECK failed" | sed 's/^/checked build: JF_DCHECK format strings in the library: /' | tee gpurun_out/checked_tests.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider >> gpurun_out/checked_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/checked_tests.log
grep -c "JF_DCHECK failed" gpurun_out/checked_tests.log | sed 's/^/JF_DCHECK failures reported: /' >> gpurun_out/checked_tests.log
tail -5 gpurun_out/checked_tests.log

#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (GPU box).  Logs in gpurun_out/sanitize_*.log;
# copy the summaries to profiles/.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_${tool}.log >> gpurun_out/sanitize_summary.txt
done
timeout 1200 $CS --tool memcheck --print-limit 20 --error-exitcode 9 python tools/sanitize_cases.py graph > gpurun_out/sanitize_memcheck_graph.log 2>&1
echo "memcheck (graph fits) rc=$?" | tee -a gpurun_out/sanitize_summary.txt
tail -3 gpurun_out/sanitize_memcheck_graph.log >> gpurun_out/sanitize_summary.txt

#!/bin/bash
# Round profile capture (run on the GPU box via gpurun).  Writes gpurun_out/:
#   bench_<tag>.json        bench.py line (no profiler attached)
#   launches_<tag>.csv      every kernel launch of a short bench run (ncu, cold, serialised)
#   jpass_<tag>.ncu-rep     ncu --set full of the T J-pass (one launch)
#   solver_<tag>.ncu-rep    ncu --set full of one solver-kernel launch
# then, here:
#   python tools/ncu_summary.py TAG gpurun_out/{jpass,solver}_TAG.ncu-rep > profiles/TAG_ncu_summary.txt
#   python tools/launch_shares.py gpurun_out/launches_TAG.csv > profiles/TAG_launch_shares.txt
set -x
TAG=${1:-r2}
WHAT=${2:-all}
mkdir -p gpurun_out
if [ "$WHAT" = all ] || [ "$WHAT" = bench ]; then
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph --no-batch > /dev/null 2>&1
fi
EXTRA=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
timeout 600 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:moment_stream -s 3 -c 1 \
    -o gpurun_out/jpass_${TAG} -f python tools/quick_time.py 4096 passonly > /dev/null 2>&1
# (fits of the moment J-passes run the solver step in the pass's last block,
# R37: the bench launches no solver kernel to capture)
ls -la gpurun_out

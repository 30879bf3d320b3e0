#!/bin/bash
# ncu --set full of the C3 (1024^2) J-pass and of a C3 fit's kernels (GPU box).
mkdir -p gpurun_out
EXTRA=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
timeout 600 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:moment_stream -s 3 -c 1 \
    -o gpurun_out/jpass_c3 -f python tools/quick_time.py 1024 passonly > /dev/null 2>&1
timeout 600 python tools/sweep.py --out gpurun_out/sweep_r2.json > gpurun_out/sweep_r2.log 2>&1
tail -3 gpurun_out/sweep_r2.log

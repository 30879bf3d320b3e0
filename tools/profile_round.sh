#!/bin/bash
# Round profile capture (run on the GPU box via gpurun).  Writes gpurun_out/:
#   bench_<tag>.json        bench.py line (no profiler attached)
#   launches_<tag>.csv      every kernel launch of a short bench run (ncu, cold, serialised)
#   jpass_<tag>.ncu-rep     ncu --set full of the T J-pass (one launch)
#   rpass_<tag>.ncu-rep     ncu --set full of the T r-pass (one launch)
#   solver_<tag>.ncu-rep    ncu --set full of one solver-kernel launch
# then, here:
#   python tools/ncu_summary.py TAG gpurun_out/{jpass,rpass,solver}_TAG.ncu-rep > profiles/TAG_ncu_summary.txt
#   python tools/launch_shares.py gpurun_out/launches_TAG.csv > profiles/TAG_launch_shares.txt
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moment_ -s 3 -c 1 \
    -o gpurun_out/jpass_${TAG} -f python tools/quick_time.py 4096 passonly > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^pass_kernel -s 3 -c 1 \
    -o gpurun_out/rpass_${TAG} -f python tools/quick_time.py 4096 passonly > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solver_kernel -s 20 -c 1 \
    -o gpurun_out/solver_${TAG} -f python tools/quick_time.py 4096 > /dev/null 2>&1
ls -la gpurun_out

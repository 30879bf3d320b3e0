#!/bin/bash
# Development aid (GPU box): JF_DEV build (per-warp globaltimer stamps), then
# the per-warp timeline of one moment J-pass at W (tools/stamps2.py).
W=${1:-4096}
mkdir -p gpurun_out
nproc
JF_DEV=1 python -m paper_2208_12187_b200.build --force > gpurun_out/devbuild.log 2>&1 || { tail -30 gpurun_out/devbuild.log; exit 1; }
JF_DEBUG_STAMPS=/tmp/st.bin python tools/quick_time.py $W passonly
python tools/stamps2.py /tmp/st.bin

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
TRACE_SO=tools/ab/libgi_trace.so timeout 600 python tools/trace_async.py cfg4 2 bsp > gpurun_out/r02e_trace_cfg4.txt 2>&1
python tools/profile_run.py --config 4 --delta 2 --reps 2 > gpurun_out/r02e_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 1 -c 1 -o gpurun_out/r02e_cfg4 -f \
  python tools/profile_run.py --config 4 --delta 2 --reps 2 > gpurun_out/r02e_ncu.log 2>&1

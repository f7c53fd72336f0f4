#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
for d in 32768 65536 131072 262144 524288; do timeout 300 python tools/time_cfg.py 2 $d '{}'; done > gpurun_out/r02af_delta.log 2>&1
TRACE_SO=tools/ab/libgi_trace.so timeout 600 python tools/trace_async.py cfg2 65536 bsp > gpurun_out/r02af_trace_cfg2.txt 2>&1

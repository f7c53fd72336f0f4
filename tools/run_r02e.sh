#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
TRACE_W=1024 TRACE_SO=tools/ab/libgi_trace1024.so timeout 600 python tools/trace_async.py cfg4 2 bsp > gpurun_out/r02e_trace_cfg4.log 2>&1
TRACE_W=1024 TRACE_SO=tools/ab/libgi_trace1024.so timeout 600 python tools/trace_async.py cfg4 2 unfused > gpurun_out/r02e_trace_cfg4u.log 2>&1
timeout 900 python tools/time_cfg.py 4 2 '{}' '{"fusion": false}' '{"threshold": 64}' '{"threshold": 1024}' '{"threshold": 2048}' > gpurun_out/r02e_cfg4_T.log 2>&1

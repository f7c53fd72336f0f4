#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
TRACE_SO=tools/ab/libgi_trace.so timeout 600 python tools/trace_async.py cfg4 2 bsp > gpurun_out/r02g_trace_cfg4.txt 2>&1

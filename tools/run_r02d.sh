#!/bin/bash
# traces of config 4 (1024 threads) and config 2 (512), and the config-5 batch Δ / shape sweep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
TRACE_W=1024 TRACE_SO=tools/ab/libgi_trace1024.so timeout 600 python tools/trace_async.py cfg4 2 bsp > gpurun_out/r02d_trace_cfg4.log 2>&1
TRACE_W=512 TRACE_SO=tools/ab/libgi_trace512.so timeout 600 python tools/trace_async.py cfg2 65536 bsp > gpurun_out/r02d_trace_cfg2.log 2>&1
timeout 900 python tools/batch_sweep.py 4096,8192,16384,32768,65536 '{}' > gpurun_out/r02d_batch_delta.log 2>&1
timeout 600 python tools/batch_sweep.py 8192 '{"cta_threads": 512}' '{"group_ctas": 4, "cta_threads": 512}' '{"rung": 3}' > gpurun_out/r02d_batch_shape.log 2>&1

#!/bin/bash
# round-2 experiment A: config-4 phase profile (GI_TRACE) and L2 eviction-policy variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
nproc > gpurun_out/r02a_host.txt; free -g >> gpurun_out/r02a_host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/r02a_host.txt
python -c "import sys; sys.path.insert(0,'.'); import gen, time; t=time.time(); gen.config_graph(4); gen.config_graph(3); print('gen', time.time()-t)" > gpurun_out/r02a_gen.txt 2>&1
for v in base ef el efel; do AB_ONLY=$v timeout 300 python tools/ab_time.py 4 2; done > gpurun_out/r02a_ab4.txt 2>&1
for v in base ef el efel; do AB_ONLY=$v timeout 300 python tools/ab_time.py 3 2; done > gpurun_out/r02a_ab3.txt 2>&1
TRACE_SO=tools/ab/libgi_trace.so timeout 600 python tools/trace_async.py cfg4 2 bsp > gpurun_out/r02a_trace_cfg4.txt 2>&1
TRACE_SO=tools/ab/libgi_trace.so timeout 300 python tools/trace_async.py cfg3 2 bsp > gpurun_out/r02a_trace_cfg3.txt 2>&1

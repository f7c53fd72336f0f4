#!/bin/bash
# round 2 (session 4): stage-A warp skip A/B (tools/abx/libgi_{base,wskip}.so) and the finer cfg2 level trace
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
TRACE_W=512 TRACE_SO=$GRAFT_REPO_ROOT/tools/abx/libgi_trace512.so timeout 600 python tools/trace_async.py cfg2 65536 bsp > gpurun_out/r02o_trace_cfg2.log 2>&1
for r in 1 2; do for v in base wskip; do
  for cd in "2 65536" "1 1000" "3 2" "5 8192"; do
    AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02o_ab.log
  done
done; done
for v in base wskip; do AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02o_ab.log; done

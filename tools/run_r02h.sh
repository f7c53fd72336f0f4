#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
for r in 1 2; do for v in base l1; do
  AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 >> gpurun_out/r02h_ab4.log 2>&1
done; done
for v in base l1; do AB_ONLY=$v timeout 600 python tools/ab_time.py 3 2 >> gpurun_out/r02h_ab3.log 2>&1; done

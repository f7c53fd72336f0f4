#!/bin/bash
# round 2 (session 4): slot-load L2 policy A/B on every config (c0 = the mirror commit's build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in c0 ef0 ef1; do
  for cd in "4 2" "2 65536" "5 8192" "3 2"; do
    AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02s_ab.log
  done
done; done

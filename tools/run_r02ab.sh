#!/bin/bash
# round 2 (session 4): extraction dist reads with an L2 evict-first policy (A/B on configs 4 and 3)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in xd0 xd1; do
  for cd in "4 2" "3 2" "2 65536"; do AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02ab_ab.log; done
done; done

#!/bin/bash
# round 2 (session 4): L2 policies for the wavefront's dist lines vs the slot stream (A/B)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in base el ef elef persist; do
  for cd in "2 65536" "1 1000" "5 8192" "3 2"; do
    if [ $v = persist ]; then
      GI_L2_PERSIST=1 AB_ONLY=base timeout 600 python tools/ab_time.py $cd 2>&1 | grep -E "libgi|L2 window" | sed "s/^/cfg $cd persist: /" >> gpurun_out/r02p_ab.log
    else
      AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02p_ab.log
    fi
  done
done; done

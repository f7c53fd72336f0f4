#!/bin/bash
# round 2 (session 4): k-core slot path — warp match vs one atomic per edge, slot evict-first (A/B)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export AB_DIR=abx
for r in 1 2; do for v in kb knm kef knmef; do
  for c in 2 1; do AB_ONLY=$v timeout 600 python tools/ab_kcore.py $c 2>&1 | grep libgi | sed "s/^/cfg $c: /" >> gpurun_out/r02z_ab.log; done
done; done

#!/bin/bash
# round 2 (session 4): expand rows-in-flight sweep (kXRows) with the mirror, and a --set full
# capture of config 4's hub-phase expand_kernel (the second expand launch of the query)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
for r in 1 2; do for v in xr4 xr8 xr12 xr16; do
  AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4: /" >> gpurun_out/r02u_ab.log
done; done
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 1 -c 1 -o gpurun_out/r02u_expand -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02u_ncu.log 2>&1

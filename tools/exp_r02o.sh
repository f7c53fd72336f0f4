#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02o_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 1 -c 1 -o gpurun_out/r02o_expand -f \
  python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02o_ncu.log 2>&1

#!/bin/bash
# round-2 experiment B: ncu --set full of the config-4 query (source-level stalls)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 2 > gpurun_out/r02b_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 1 -c 1 -o gpurun_out/r02b_cfg4 -f \
  python tools/profile_run.py --config 4 --delta 2 --reps 2 > gpurun_out/r02b_ncu.log 2>&1

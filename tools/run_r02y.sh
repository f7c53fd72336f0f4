#!/bin/bash
# round 2 (session 4): --set full captures of config 4's persistent segments (the post-hub-phase
# segment and the tail segment) for the stall and traffic breakdown
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 5 -c 1 -o gpurun_out/r02y_seg5 -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 17 -c 1 -o gpurun_out/r02y_seg17 -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_ncu17.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:extract_kernel -s 1 -c 1 -o gpurun_out/r02y_extract -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02y_ncux.log 2>&1

#!/bin/bash
# round-2 profiles of the config-4 headline: the bench launch list (time + DRAM bytes per launch),
# then ncu --set full of the hub-phase expand_kernel and the heaviest persistent segment
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary --no-compare"
$CMD > gpurun_out/r02ad_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand" --csv --log-file gpurun_out/r02ad_launches.csv $CMD > gpurun_out/r02ad_ncu1.log 2>&1
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ad_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 1 -c 1 -o gpurun_out/r02ad_expand -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ad_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sssp_persistent -s 3 -c 1 -o gpurun_out/r02ad_persist -f python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02ad_ncu3.log 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 2 > gpurun_out/r02n_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r02n_launches.csv python tools/profile_run.py --config 4 --delta 2 --reps 2 > gpurun_out/r02n_ncu.log 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02p_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_requests_srcunit_tex_op_atom.sum --clock-control none -k regex:"sssp|expand" --csv --log-file gpurun_out/r02p_launches.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02p_ncu.log 2>&1

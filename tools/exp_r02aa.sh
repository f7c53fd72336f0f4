#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expand or hubs" > gpurun_out/r02aa_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02aa_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"expand": "on"}' > gpurun_out/r02aa_time4.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"expand": "on"}' > gpurun_out/r02aa_time3.log 2>&1
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02aa_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"sssp|expand" --csv --log-file gpurun_out/r02aa_launches.csv python tools/time_cfg.py 4 2 '{"expand": "on", "reps": 1}' > gpurun_out/r02aa_ncu.log 2>&1

#!/bin/bash
# round 2 (session 4): mirror test, config-4 launch list with DRAM bytes (mirror on), config-2 level trace
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mirror" > gpurun_out/r02n_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02n_tests.log
python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02n_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/r02n_launches.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02n_ncu1.log 2>&1
TRACE_W=512 timeout 900 python tools/trace_async.py cfg2 65536 bsp > gpurun_out/r02n_trace_cfg2.log 2>&1

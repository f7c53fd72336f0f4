#!/bin/bash
# round-2 (session 2) check: GPU tests, default bench, config-4 launch list with DRAM bytes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02c_tests.log
( time timeout 1500 python bench.py ) > gpurun_out/r02c_bench.log 2> gpurun_out/r02c_bench.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary --no-compare"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand" --csv --log-file gpurun_out/r02c_launches.csv $CMD > gpurun_out/r02c_ncu1.log 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not config4 and not config5 and not config2" > gpurun_out/r02y_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02y_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"expand": "on"}' > gpurun_out/r02y_time4.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"expand": "on"}' > gpurun_out/r02y_time3.log 2>&1
timeout 600 python tools/time_cfg.py 2 65536 '{}' > gpurun_out/r02y_time2.log 2>&1
timeout 600 python tools/time_cfg.py 1 1000 '{}' > gpurun_out/r02y_time1.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02y_bench.log 2> gpurun_out/r02y_bench.err
echo "bench rc=$?" >> gpurun_out/r02y_bench.err

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expand or hubs" > gpurun_out/r02ab_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ab_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"expand": "on"}' > gpurun_out/r02ab_time4.log 2>&1
for sm in 1000000 16000000 64000000; do GI_SPLIT_MIN=$sm timeout 600 python tools/time_cfg.py 4 2 '{"expand": "on"}'; done > gpurun_out/r02ab_time4_sm.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"expand": "on"}' > gpurun_out/r02ab_time3.log 2>&1
for sm in 1000000 16000000; do GI_SPLIT_MIN=$sm timeout 600 python tools/time_cfg.py 3 2 '{"expand": "on"}'; done > gpurun_out/r02ab_time3_sm.log 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expand or hubs" > gpurun_out/r02f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02f_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"expand": "off"}' > gpurun_out/r02f_time4.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"expand": "off"}' > gpurun_out/r02f_time3.log 2>&1

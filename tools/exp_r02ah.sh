#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expand or hubs or config3 or lazy" > gpurun_out/r02ah_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ah_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"cta_threads": 512}' '{"expand": "off"}' > gpurun_out/r02ah_time4.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' > gpurun_out/r02ah_time3.log 2>&1
timeout 600 python tools/time_cfg.py 2 65536 '{}' > gpurun_out/r02ah_time2.log 2>&1

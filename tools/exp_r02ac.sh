#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not config2 and not config5" > gpurun_out/r02ac_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ac_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"expand": "off"}' > gpurun_out/r02ac_time4.log 2>&1
for sm in 262144 4000000; do GI_SPLIT_MIN=$sm timeout 600 python tools/time_cfg.py 4 2 '{}'; done > gpurun_out/r02ac_time4_sm.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"expand": "on"}' > gpurun_out/r02ac_time3.log 2>&1

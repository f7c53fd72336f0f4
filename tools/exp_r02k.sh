#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not config4 and not config5 and not config2" > gpurun_out/r02k_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02k_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"cta_threads": 512}' '{"expand": "off"}' > gpurun_out/r02k_time4.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"cta_threads": 512}' '{"expand": "off"}' > gpurun_out/r02k_time3.log 2>&1
timeout 600 python tools/time_cfg.py 2 65536 '{}' '{"drain": "async"}' > gpurun_out/r02k_time2.log 2>&1
timeout 600 python tools/time_cfg.py 1 1000 '{}' > gpurun_out/r02k_time1.log 2>&1

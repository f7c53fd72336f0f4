#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expand or hubs or config3 or hand or random or spec" > gpurun_out/r02x_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02x_tests.log
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"cta_threads": 512}' '{"expand": "off"}' '{"expand": "off", "cta_threads": 512}' > gpurun_out/r02x_time4.log 2>&1
GI_PAD_MB=256 timeout 600 python tools/time_cfg.py 4 2 '{}' '{"cta_threads": 512}' '{"expand": "off"}' '{"expand": "off", "cta_threads": 512}' > gpurun_out/r02x_time4_pad.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"cta_threads": 512}' '{"expand": "off"}' > gpurun_out/r02x_time3.log 2>&1
timeout 600 python tools/time_cfg.py 2 65536 '{}' > gpurun_out/r02x_time2.log 2>&1
timeout 600 python tools/time_cfg.py 1 1000 '{}' > gpurun_out/r02x_time1.log 2>&1

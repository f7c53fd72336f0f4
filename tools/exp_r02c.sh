#!/bin/bash
# round-2 experiment C: expand path parity + timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expand or hubs or hand or spec or random or config3 or config1" > gpurun_out/r02c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02c_tests.log
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"expand": "off"}' '{"fusion": false}' > gpurun_out/r02c_time3.log 2>&1
timeout 600 python tools/time_cfg.py 4 2 '{}' '{"expand": "off"}' '{"fusion": false}' > gpurun_out/r02c_time4.log 2>&1
GI_PACK=0 timeout 600 python tools/time_cfg.py 4 2 '{}' > gpurun_out/r02c_time4_nopack.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config4" > gpurun_out/r02c_cfg4.log 2>&1
echo "cfg4 rc=$?" >> gpurun_out/r02c_cfg4.log

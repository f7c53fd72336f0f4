#!/bin/bash
# extraction split: parity (new test + split tests + config 4 full), timing on config 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "extract_split or expand_split or expand_edge or hand_examples or lazy or config3_full" > gpurun_out/r02f_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_tests.log
timeout 900 python tools/time_cfg.py 4 2 '{}' '{"fusion": false}' '{"threshold": 1024}' > gpurun_out/r02f_cfg4.log 2>&1
GI_XSPLIT_MIN=0 timeout 600 python tools/time_cfg.py 4 2 '{}' > gpurun_out/r02f_cfg4_nox.log 2>&1
GI_XSPLIT_MIN=500000 timeout 600 python tools/time_cfg.py 4 2 '{}' > gpurun_out/r02f_cfg4_x500k.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config4_full" > gpurun_out/r02f_cfg4_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_cfg4_parity.log

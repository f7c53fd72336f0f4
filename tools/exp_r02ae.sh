#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "lazy or peers_two or stress or ppsp_astar_config2 or capi" > gpurun_out/r02ae_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ae_tests.log
timeout 600 python tools/time_cfg.py 2 65536 '{}' '{"fusion": false}' '{"fusion": false, "lazy": true}' > gpurun_out/r02ae_time2.log 2>&1
timeout 600 python tools/time_cfg.py 2 1024 '{}' '{"fusion": false}' '{"fusion": false, "lazy": true}' > gpurun_out/r02ae_time2b.log 2>&1

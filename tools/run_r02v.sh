#!/bin/bash
# round 2 (session 4): batched host segment loop (speculative [expand, extract, resume] rounds)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand or ppsp or astar or stress" > gpurun_out/r02v_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02v_tests.log
tail -3 gpurun_out/r02v_tests.log
for r in 1 2 3; do timeout 600 python tools/time_cfg.py 4 2 '{}' '{"fusion": false}' 2>&1 | grep ms_median | cut -c1-300 >> gpurun_out/r02v_cfg4.log; done

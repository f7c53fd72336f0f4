#!/bin/bash
# round 2 (session 4): bucket window — parity of the split/window paths, then config 4 per width
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand" > gpurun_out/r02r_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02r_tests.log
tail -3 gpurun_out/r02r_tests.log
for r in 1 2; do for w in 0 4 8 16; do
  GI_WINDOW=$w timeout 600 python tools/time_cfg.py 4 2 '{}' 2>&1 | grep ms_median | sed "s/^/window=$w /" >> gpurun_out/r02r_ab4.log
done; done

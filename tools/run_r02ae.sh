#!/bin/bash
# round 2 (session 4): the bucket window opened late (GI_WINDOW_PILE) — tests, config 4 A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window" > gpurun_out/r02ae_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ae_tests.log
tail -2 gpurun_out/r02ae_tests.log
for r in 1 2; do for wp in "0 0" "4 2000000" "4 8000000" "8 4000000" "2 1000000"; do
  set -- $wp
  GI_WINDOW=$1 GI_WINDOW_PILE=$2 timeout 600 python tools/time_cfg.py 4 2 '{}' 2>&1 | grep ms_median | cut -c1-330 | sed "s/^/window=$1 pile=$2 /" >> gpurun_out/r02ae_ab.log
done; done

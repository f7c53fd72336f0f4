#!/bin/bash
# round 2 (session 4): the persistent kernel's pre-reads through the expand mirror — tests, A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "window or mirror or split or expand or stress or ppsp or astar or hubs" > gpurun_out/r02ac_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ac_tests.log
tail -2 gpurun_out/r02ac_tests.log
for r in 1 2; do for v in pm0 pm1; do
  AB_ONLY=$v timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg 4: /" >> gpurun_out/r02ac_ab.log
done; done

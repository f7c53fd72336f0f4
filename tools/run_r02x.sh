#!/bin/bash
# round 2 (session 4): the parent-edge skip of the low-degree fused kernels — GPU tests, then A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx
GI_SKIP_CFG4=1 timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02x_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02x_tests.log
tail -3 gpurun_out/r02x_tests.log
for r in 1 2; do for v in par0 par1; do
  for cd in "2 65536" "1 1000" "5 8192" "2 16384"; do
    AB_ONLY=$v timeout 600 python tools/ab_time.py $cd 2>&1 | grep libgi | sed "s/^/cfg $cd: /" >> gpurun_out/r02x_ab.log
  done
done; done

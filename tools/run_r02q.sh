#!/bin/bash
# round 2 (session 4): expand fast block path + 32-bit edge positions (A/B on config 4), split-path parity
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache AB_DIR=abx2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mirror or split or expand" > gpurun_out/r02q_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02q_tests.log
for r in 1 2; do
  GI_IDX32=0 AB_ONLY=fb0 timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4 fb0 idx64: /" >> gpurun_out/r02q_ab.log
  AB_ONLY=fb0 timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4 fb0 idx32: /" >> gpurun_out/r02q_ab.log
  AB_ONLY=fb1 timeout 600 python tools/ab_time.py 4 2 2>&1 | grep libgi | sed "s/^/cfg4 fb1 idx32: /" >> gpurun_out/r02q_ab.log
done

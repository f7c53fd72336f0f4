#!/bin/bash
# round 2 (session 4): expand's mirror filter — parity of the split paths, then config 4 A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mirror or split or expand" > gpurun_out/r02m_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02m_tests.log
for r in 1 2; do for mv in 1 0; do
  GI_MIRROR=$mv timeout 600 python tools/time_cfg.py 4 2 '{}' >> gpurun_out/r02m_ab4.log 2>&1; echo "mirror=$mv" >> gpurun_out/r02m_ab4.log
done; done

#!/bin/bash
# GPU tests after the cluster-flag fix, the fusion-threshold sweep and the eager/lazy table
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02b_tests.log
timeout 900 python tools/sweep_T.py 1 2 3 > gpurun_out/r02b_sweepT.md 2>&1
timeout 900 python tools/lazy_table.py 1 2 3 4 > gpurun_out/r02b_lazy.md 2>&1

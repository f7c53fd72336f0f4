#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "kcore" > gpurun_out/r02g_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02g_tests.log
for c in 2 3 1; do
  timeout 300 python tools/profile_run.py --config $c --kcore --reps 5 > gpurun_out/r02g_kc$c.log 2>&1
  GI_KC_SLOTS=0 timeout 300 python tools/profile_run.py --config $c --kcore --reps 5 > gpurun_out/r02g_kc${c}_csr.log 2>&1
done
timeout 300 python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02g_plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sssp|expand|extract" --csv --log-file gpurun_out/r02g_launches4.csv python tools/profile_run.py --config 4 --delta 2 --reps 1 > gpurun_out/r02g_ncu4.log 2>&1

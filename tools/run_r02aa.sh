#!/bin/bash
# round 2 (session 4): k-core — slot path without the warp match + evict-first slots (now default),
# packed 4-byte edges on the CSR path (GI_KC_PACK=0: the 8-byte edges); k-core parity tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export AB_DIR=abm AB_ONLY=main
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "kcore" > gpurun_out/r02aa_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02aa_tests.log
tail -2 gpurun_out/r02aa_tests.log
for r in 1 2; do for pk in 1 0; do
  GI_KC_PACK=$pk timeout 600 python tools/ab_kcore.py 3 2>&1 | grep libgi | sed "s/^/cfg 3 pack=$pk: /" >> gpurun_out/r02aa_ab.log
done; done
timeout 600 python tools/ab_kcore.py 2 2>&1 | grep libgi | sed "s/^/cfg 2: /" >> gpurun_out/r02aa_ab.log

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "hand or spec or random or config1 or path or async or drain or lazy or ppsp or astar or peers_one or single_cta or threads" > gpurun_out/r02ag_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02ag_tests.log
python -c "import sys; sys.path.insert(0,'.'); import gen; gen.config_graph(2)"
for v in quad octet quad octet; do AB_ONLY=$v timeout 300 python tools/ab_time.py 2 65536; done > gpurun_out/r02ag_ab2.txt 2>&1
for v in quad octet; do AB_ONLY=$v timeout 300 python tools/ab_time.py 1 1000; done > gpurun_out/r02ag_ab1.txt 2>&1
for v in quad octet; do AB_ONLY=$v timeout 300 python tools/ab_time.py 5 8192; done > gpurun_out/r02ag_ab5.txt 2>&1

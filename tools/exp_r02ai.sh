#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python -c "import sys; sys.path.insert(0,'.'); import gen; gen.config_graph(4)"
for v in base xtr8 xr4 xr12 base; do AB_ONLY=$v timeout 300 python tools/ab_time.py 4 2; done > gpurun_out/r02ai_ab4.txt 2>&1
for v in base xtr8; do AB_ONLY=$v AB_OPTS=cta_threads=512 timeout 300 python tools/ab_time.py 4 2; done >> gpurun_out/r02ai_ab4.txt 2>&1
for v in base xtr8; do AB_ONLY=$v timeout 300 python tools/ab_time.py 3 2; done > gpurun_out/r02ai_ab3.txt 2>&1

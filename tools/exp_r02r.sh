#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python -c "import sys; sys.path.insert(0,'.'); import gen; gen.config_graph(4)"
for v in cs ldg ncpol; do AB_ONLY=$v timeout 300 python tools/ab_time.py 4 2; done > gpurun_out/r02r_ab4.txt 2>&1

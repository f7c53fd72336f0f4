#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python -c "import sys; sys.path.insert(0,'.'); import gen; gen.config_graph(4)"
( for p in -1 0 256 512; do PAD_MB=$p python tools/gather_probe.py; done ) 2>&1 | grep -v Warn > gpurun_out/r02w_gather_pad.txt

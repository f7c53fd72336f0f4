#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python -c "import sys; sys.path.insert(0,'.'); import gen; gen.config_graph(4)"
timeout 600 python tools/stream_probe.py 4 2 > gpurun_out/r02s_stream4.txt 2>&1
timeout 600 python tools/stream_probe.py 2 65536 > gpurun_out/r02s_stream2.txt 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python -c "import sys; sys.path.insert(0,'.'); import gen; gen.config_graph(4); gen.config_graph(1)"
( echo chunked; timeout 300 python tools/placement_test.py single; echo chunked; timeout 300 python tools/placement_test.py single;
  echo cudamalloc; GI_CHUNK_DIST=0 timeout 300 python tools/placement_test.py single;
  echo chunked-pad512; GI_PAD_MB=512 timeout 300 python tools/placement_test.py single ) > gpurun_out/r02t_chunk.txt 2>&1
timeout 600 python tools/time_cfg.py 2 65536 '{}' > gpurun_out/r02t_time2.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"expand": "off"}' > gpurun_out/r02t_time3.log 2>&1

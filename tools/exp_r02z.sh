#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
GI_DUMP_X=/tmp/xdump timeout 600 python tools/time_cfg.py 4 2 '{"expand": "on", "reps": 1}' > gpurun_out/r02z_dump.log 2>&1
ls -la /tmp/xdump* > gpurun_out/r02z_files.txt
XDUMP=/tmp/xdump python tools/relax_probe.py > gpurun_out/r02z_relax.log 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/gather_probe.py > gpurun_out/r02i_gather.log 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
python tools/relax_probe.py > gpurun_out/r02j_relax.log 2>&1

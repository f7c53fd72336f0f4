#!/bin/bash
# round 2 (session 4): config-5 batch group shapes (CTAs per group, threads per CTA, rung) at Δ=2^13
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python tools/batch_sweep.py 8192 '{}' '{"group_ctas": 1}' '{"group_ctas": 2}' '{"group_ctas": 4}' \
  '{"group_ctas": 2, "cta_threads": 512}' '{"group_ctas": 4, "cta_threads": 512}' '{"group_ctas": 1, "cta_threads": 512}' \
  '{"group_ctas": 2, "threshold": 4096}' '{"group_ctas": 2, "threshold": 1024}' '{"group_ctas": 2, "rung": "grid"}' > gpurun_out/r02w_batch.log 2>&1

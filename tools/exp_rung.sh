#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export GI_GEN_CACHE=/tmp/gcache
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "rungs or hand or path or capi" > gpurun_out/rung_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rung_tests.log
timeout 600 python tools/time_cfg.py 1 1000 '{}' '{"rung": "cta"}' '{"rung": "cluster", "group_ctas": 4}' '{"rung": "cluster", "group_ctas": 8}' '{"rung": "cluster", "group_ctas": 16}' '{"max_ctas": 16}' > gpurun_out/rung_time1.log 2>&1
timeout 600 python tools/time_cfg.py 2 65536 '{}' '{"rung": "cluster", "group_ctas": 16}' > gpurun_out/rung_time2.log 2>&1
timeout 600 python tools/time_cfg.py 3 2 '{}' '{"rung": "cluster", "group_ctas": 16}' > gpurun_out/rung_time3.log 2>&1
timeout 900 python - > gpurun_out/rung_time5.log 2>&1 <<'PY'
import sys, json, statistics; sys.path.insert(0, '.')
import torch, gen
from paper_1911_07260_b200 import gi
g = gen.config_graph(5); G = gi.Graph.from_csr(g); srcs = gen.config_sources(5, g, 64)
out = torch.empty((64, g.n), dtype=torch.int32, device="cuda")
for o in ({}, {"rung": "cta"}, {"rung": "cluster", "group_ctas": 2}, {"rung": "cluster", "group_ctas": 4}, {"group_ctas": 4}):
    ts = []
    for i in range(3):
        st = gi.gi_sssp_batch(G, srcs, 8192, out, gi.make_options(**o)); ts.append(st[0].gpu_ms)
    print(json.dumps({"opts": o, "ms": statistics.median(ts), "groups": st[0].groups, "ctas": st[0].ctas, "rung": st[0].rung}), flush=True)
PY

"""Time one config through the product library with option sets given as JSON dicts.
usage: python tools/time_cfg.py CONFIG DELTA '{"expand": "off"}' '{}' ...   (GI_GEN_CACHE speeds up cfg 3/4)"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import gen  # noqa: E402
import torch  # noqa: E402
from paper_1911_07260_b200 import gi  # noqa: E402

cfg, delta = int(sys.argv[1]), int(sys.argv[2])
sets = [json.loads(x) for x in sys.argv[3:]] or [{}]
g = gen.config_graph(cfg)
G = gi.Graph.from_csr(g)
src = gen.config_source(cfg, g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
ref = None
for o in sets:
    reps = int(o.pop("reps", 7))
    ts, st = [], None
    for i in range(reps + 2):
        st = gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**o))
        if i >= 2:
            ts.append(st.gpu_ms)
    d = gi.as_uint32(out)
    same = None if ref is None else bool(np.array_equal(d, ref))
    if ref is None:
        ref = d.copy()
    print(json.dumps({"config": cfg, "delta": delta, "opts": o, "ms_median": statistics.median(ts), "ms_min": min(ts),
                      "same_as_first": same, **{k: getattr(st, k) for k in (
                          "buckets", "rounds", "grid_syncs", "fused_subrounds", "spills", "vertices_processed",
                          "edges_relaxed", "far_scanned", "critical_subrounds", "threads_per_cta")}}), flush=True)

"""Config-5 batch (64 sources on the config-2 grid, one GPU) over Δ and option sets.
usage: python tools/batch_sweep.py DELTA[,DELTA...] '{"group_ctas": 2}' '{}' ...
Prints device ms per batch (stats[0].gpu_ms), median of 3 after 1 warm-up, with counters
summed over the 64 sources; the first run's rows are the reference for `same`."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import gen  # noqa: E402
import torch  # noqa: E402
from paper_1911_07260_b200 import gi  # noqa: E402

deltas = [int(x) for x in sys.argv[1].split(",")]
sets = [json.loads(x) for x in sys.argv[2:]] or [{}]
g = gen.config_graph(2)
G = gi.Graph.from_csr(g)
srcs = gen.config_sources(5, g)
out = torch.empty((len(srcs), g.n), dtype=torch.int32, device="cuda")
ref = None
for delta in deltas:
    for o in sets:
        o = dict(o)
        reps = int(o.pop("reps", 3))
        ts = []
        for i in range(reps + 1):
            st = gi.gi_sssp_batch(G, srcs, delta, out, gi.make_options(**o))
            if i >= 1:
                ts.append(st[0].gpu_ms)
        row0 = out[0].cpu().numpy().copy()
        same = None if ref is None else bool(np.array_equal(row0, ref))
        if ref is None:
            ref = row0
        tot = lambda k: int(sum(getattr(s, k) for s in st))
        print(json.dumps({"delta": delta, "opts": o, "ms_median": statistics.median(ts), "same_row0": same,
                          "ctas": st[0].ctas, "threads": st[0].threads_per_cta, "groups": st[0].groups,
                          "rung": getattr(st[0], "rung", None),
                          **{k: tot(k) for k in ("buckets", "rounds", "vertices_processed", "edges_relaxed",
                                                  "spills", "far_scanned")}}), flush=True)

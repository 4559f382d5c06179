"""Dev tool (GPU box): device time of a bench workload over the values of one engine option.

    python tools/option_probe.py <workload> <sources> <option> <value> [<value> ...]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2008_05718_b200._capi import Engine, MODE_DIRECT  # noqa: E402
from paper_2008_05718_b200.engine import default_groups  # noqa: E402

name, k, key = sys.argv[1], int(sys.argv[2]), sys.argv[3]
values = [int(x) for x in sys.argv[4:]]
g, label = bench.workload(name)
src = bench.pick_sources(g.num_vertices, k)
ref = None
for val in values:
    with Engine(g, 0) as e:
        e.set_option("groups", default_groups(g, len(src)))
        e.set_option("reports", 0)
        e.set_option("relabel", 1)
        e.set_option(key, val)
        e.run(src, MODE_DIRECT)
        best = None
        for rep in range(3):
            bc, st = e.run(src, MODE_DIRECT)
            if best is None or st["ms_total"] < best["ms_total"]:
                best = st
    if ref is None:
        ref = bc
    rel = float(np.max(np.abs(bc - ref) / np.maximum(np.abs(ref), 1e-300)))
    print(json.dumps({"workload": name, key: val, "ms": round(best["ms_total"], 3), "fwd": round(best["ms_forward"], 3),
                      "bwd": round(best["ms_backward"], 3), "launches": int(best["launches"]),
                      "gteps": round(g.num_edges * len(src) / best["ms_total"] / 1e6, 1), "max_rel_vs_first": rel}), flush=True)

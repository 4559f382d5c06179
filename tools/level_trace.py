"""Dev tool (GPU box): per-level launch times of one warm run (BC_LEVEL_TRACE) on a bench workload.

    python tools/level_trace.py [workload] [sources] [bwd_push]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2008_05718_b200._capi import Engine, MODE_DIRECT  # noqa: E402
from paper_2008_05718_b200.engine import default_groups  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
beta = int(sys.argv[3]) if len(sys.argv) > 3 else 4
g, label = bench.workload(name)
src = bench.pick_sources(g.num_vertices, k)
with Engine(g, 0) as e:
    e.set_option("groups", default_groups(g, len(src)))
    e.set_option("reports", 0)
    e.set_option("relabel", 1)
    e.set_option("bwd_push", beta)
    e.run(src, MODE_DIRECT)
    e.run(src, MODE_DIRECT)
    os.environ["BC_LEVEL_TRACE"] = "1"
    print("bwd_push", beta, flush=True)
    bc, st = e.run(src, MODE_DIRECT)
    print({k2: round(v, 3) for k2, v in st.items() if k2.startswith("ms_")}, flush=True)

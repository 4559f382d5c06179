"""Dev tool: gather-loop counters of one batch (needs a -DBC_PROFILE build in BC_B200_LIB)."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tune import cached_graph
from paper_2008_05718_b200._capi import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = cached_graph(name)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), 1024))
with Engine(g) as e:
    e.set_option("groups", groups)
    bc, st = e.run(srcs[:groups * 32])
print({k: st[k] for k in ("reached", "arcs_reached", "dag_arcs", "ms_forward", "ms_backward")})

"""Dev tool: one hybir batch on the road-like 2048^2 graph in 8 strips (for ncu launch lists)."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_HYBIR
side = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = G.road_like(side, side, keep=0.2, seed=1)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), 512))
part = P.strip_partition(side, side, k)
with Engine(g) as e:
    e.set_option("groups", 16)
    e.set_option("reports", 0)
    e.set_partition(k, part.assignment)
    if len(sys.argv) > 3:
        e.run(srcs[:32], MODE_HYBIR)
    bc, st = e.run(srcs, MODE_HYBIR)
    print({k_: st[k_] for k_ in ("ms_total", "ms_border", "ms_forward", "ms_backward", "iterations", "launches")})
    bc, st = e.run(srcs, MODE_HYBIR)
print({k_: st[k_] for k_ in ("ms_total", "ms_border", "ms_forward", "ms_backward", "iterations", "launches")})

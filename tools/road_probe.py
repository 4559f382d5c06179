"""Dev tool: one run of the road-like 2048x2048 graph (config 3, unpartitioned view)."""
import os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine
side = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 512
groups = int(sys.argv[3]) if len(sys.argv) > 3 else 16
opts = [o.split("=") for o in sys.argv[4:]]
g = G.road_like(side, side, keep=0.2, seed=1)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), nsrc))
with Engine(g) as e:
    e.set_option("groups", groups)
    for k, v in opts:
        e.set_option(k, int(v))
    for r in range(2):
        t0 = time.time(); bc, st = e.run(srcs); wall = time.time() - t0
    print(dict(side=side, sources=nsrc, groups=groups, opts=opts, wall_ms=round(wall * 1e3, 1), ms=round(st["ms_total"], 1),
               fwd=round(st["ms_forward"], 1), bwd=round(st["ms_backward"], 1), levels=st["max_levels"],
               launches=st["launches"], bcsum=float(bc.sum())), flush=True)

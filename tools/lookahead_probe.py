"""Step-1 look-ahead (pipeline_sources) on road-like 2048x2048 in 8 strips: time and parity against run_bc."""
import os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
side = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = G.road_like(side, side, keep=0.2, seed=1)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), 512))
part = P.strip_partition(side, side, 8)
cfg = P.RunConfig(sources=srcs, mode="hybir", partition=part, num_partitions=8, groups=groups, per_source_reports=False,
                  table_cache_dir="/tmp/bc_tables")
P.run_bc(g, cfg)                      # builds (and caches) the border tables
for name, fn in (("run_bc", P.run_bc), ("pipeline_sources", P.pipeline_sources), ("run_bc", P.run_bc),
                 ("pipeline_sources", P.pipeline_sources)):
    t0 = time.time(); res = fn(g, cfg); wall = time.time() - t0
    print(dict(call=name, groups=groups, batches=res.stats["batches"], wall_ms=round(wall * 1e3, 1),
               device_ms=round(res.stats["ms_total"], 1), border_ms=round(res.stats["ms_border"], 1),
               overlaps=res.pipeline_overlaps, cached_tables=res.stats["border_tables_from_cache"],
               bcsum=float(res.bc.sum())), flush=True)
    if name == "run_bc":
        ref = res.bc
    else:
        print("   identical to run_bc:", bool(np.array_equal(ref, res.bc)), flush=True)

"""Dev tool: does grouping sources by their distance profile to the top hubs beat the 2-hop key?"""
import json, os, random, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tune import cached_graph
from paper_2008_05718_b200._capi import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
g = cached_graph(name)
srcs = np.array(sorted(random.Random(0).sample(range(g.num_vertices), nsrc)))
deg = np.diff(g.offsets)

def timeit(e, order, tag):
    e.run(list(order[:512]))
    best = None
    for rep in range(3):
        bc, st = e.run(list(order))
        if best is None or st["ms_total"] < best["ms_total"]:
            best = st
    print(json.dumps(dict(tag=tag, ms=round(best["ms_total"], 2), fwd=round(best["ms_forward"], 2),
                          bwd=round(best["ms_backward"], 2), bcsum=float(bc.sum()))), flush=True)

with Engine(g) as e:
    e.set_option("groups", 16)
    timeit(e, srcs, "engine 2-hop key")
    e.set_option("reorder", 0)
    live = srcs[deg[srcs] > 0]
    dead = srcs[deg[srcs] == 0]
    timeit(e, np.concatenate([live, dead]), "caller order (isolated last)")
    for nh in (4, 8, 16, 32):
        hubs = np.argsort(-deg)[:nh]
        dist, _, _ = e.debug_sources(list(hubs), want=("dist",))
        d = dist[:, live].astype(np.int64)          # [hub][source]
        d[d < 0] = 7
        d = np.minimum(d, 7)
        key = np.zeros(len(live), dtype=np.uint64)
        for j in range(nh):                          # top hub in the most significant bits
            key = (key << np.uint64(2)) | np.minimum(d[j], 3).astype(np.uint64)
        order = live[np.argsort(key, kind="stable")]
        timeit(e, np.concatenate([order, dead]), "hub profile, %d hubs" % nh)
        # profile first, 2-hop key inside equal profiles
        k2 = np.array([deg[g.col_idx[g.offsets[s]:g.offsets[s + 1]]].sum() for s in live])
        order2 = live[np.lexsort((-k2, key))]
        timeit(e, np.concatenate([order2, dead]), "hub profile %d + 2-hop" % nh)
        # eccentricity-like: sum of distances to hubs, then 2-hop
        order3 = live[np.lexsort((-k2, d.sum(axis=0)))]
        timeit(e, np.concatenate([order3, dead]), "hub distance sum %d + 2-hop" % nh)

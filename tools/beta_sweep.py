"""Dev tool: push/pull threshold sweep on the bench workload."""
import json, os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tune import cached_graph
from paper_2008_05718_b200._capi import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
betas = [tuple(int(y) for y in x.split(":")) for x in (sys.argv[2] if len(sys.argv) > 2 else "4:24").split(",")]
nsrc = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
groups = int(sys.argv[4]) if len(sys.argv) > 4 else 16
g = cached_graph(name)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), nsrc))
with Engine(g) as e:
    e.set_option("groups", groups)
    for beta, late in betas:
        e.set_option("push_beta", beta)
        e.set_option("push_beta_late", late)
        e.run(srcs[:groups * 32])
        best = None
        for rep in range(3):
            bc, st = e.run(srcs)
            if best is None or st["ms_total"] < best["ms_total"]:
                best = st
        print(json.dumps(dict(beta=beta, late=late, ms=round(best["ms_total"], 2), fwd=round(best["ms_forward"], 2),
                              bwd=round(best["ms_backward"], 2), launches=best["launches"],
                              gteps=round(g.num_edges * nsrc / best["ms_total"] / 1e6, 1), bcsum=float(bc.sum()))), flush=True)

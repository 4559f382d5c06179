"""Dev tool: L1 allocation of the row gathers, whole run (row_cache) and level by level (row_bypass_mask)."""
import json, os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tune import cached_graph
from paper_2008_05718_b200._capi import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 32
g = cached_graph(name)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), 1024))
masks = [("auto", None)] + [("fwd L%d" % L, 1 << L) for L in (3, 4, 5)] + [("bwd L%d" % L, 1 << (16 + L)) for L in (1, 2, 3, 4, 5)]
for label, mask in masks:
    with Engine(g) as e:
        e.set_option("groups", groups)
        if mask is not None:
            # bit 31 keeps the mask non-zero so that every other level allocates as usual
            e.set_option("row_cache", 1); e.set_option("row_bypass_mask", mask | (1 << 31))
        e.run(srcs[:groups * 32])
        best = min((e.run(srcs)[1] for _ in range(2)), key=lambda st: st["ms_total"])
    print(json.dumps(dict(graph=name, bypass=label, ms=round(best["ms_total"], 2), fwd=round(best["ms_forward"], 2), bwd=round(best["ms_backward"], 2))), flush=True)

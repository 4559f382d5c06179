import json, os, random, sys
sys.path.insert(0, os.getcwd())
from tools.tune import cached_graph
from paper_2008_05718_b200._capi import Engine
for name, groups in (("rmat20", 32), ("er22", 8), ("rmat22", 8)):
    g = cached_graph(name)
    srcs = sorted(random.Random(0).sample(range(g.num_vertices), 1024))
    for rc in (-1, 1, 0):
        with Engine(g) as e:
            e.set_option("groups", groups); e.set_option("row_cache", rc)
            e.run(srcs[:groups * 32])
            best = min((e.run(srcs)[1] for _ in range(2)), key=lambda st: st["ms_total"])
        print(json.dumps(dict(graph=name, row_cache=rc, ms=round(best["ms_total"], 2), fwd=round(best["ms_forward"], 2), bwd=round(best["ms_backward"], 2))), flush=True)

"""More orderings (dev probe): hubs by degree, the rest grouped by their strongest hub neighbour."""
import os, sys, time, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "relabel_probe2.py")).read().split("bc0 = run(")[0])

def run(gr, sources, label):
    with Engine(gr) as e:
        e.set_option("groups", 32); e.set_option("relabel", 0)
        e.run(sources)
        best = 1e9
        for _ in range(3):
            bc, st = e.run(sources)
            best = min(best, st["ms_total"])
    print("%-60s %.2f ms  level %.2f ms" % (label, best, st["ms_level"]), flush=True)
    return bc

d_order = np.argsort(-deg, kind="stable")
rank = np.empty(n, dtype=np.int64); rank[d_order] = np.arange(n)          # degree rank (0 = biggest hub)
# strongest neighbour = neighbour with the smallest degree rank
arc_src = np.repeat(np.arange(n), deg)
best_nb = np.full(n, n, dtype=np.int64)
np.minimum.at(best_nb, arc_src, rank[col])
for T in (64, 16):
    hub = deg > T
    key1 = np.where(hub, rank, n + best_nb)             # hubs first by degree, then the rest by their strongest hub
    order = np.lexsort((rank, key1))
    gr, new_of_old = relabel(order, True)
    run(gr, sorted(new_of_old[srcs].tolist()), "hubs > %d by degree, rest grouped by strongest neighbour" % T)
gr, new_of_old = relabel(d_order, True)
run(gr, sorted(new_of_old[srcs].tolist()), "degree descending")

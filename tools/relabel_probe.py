"""Does relabelling vertices by descending degree help the dense pull kernels?  (dev probe, GPU box)
Runs the bench workload (R-MAT s20 x 1024 sources) on the graph as generated and on the relabelled
graph, same sources, and compares device time and BC (un-permuted)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine
import random

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = G.rmat(scale, 16, 1)
n = g.num_vertices
srcs = sorted(random.Random(0).sample(range(n), 1024))
deg = np.diff(g.offsets)

def relabel(g, order):
    """order[new] = old"""
    n = g.num_vertices
    new_of_old = np.empty(n, dtype=np.int64); new_of_old[order] = np.arange(n)
    src = new_of_old[g.arc_src]; dst = new_of_old[g.arc_dst]
    keep = src < dst
    return P.from_edge_arrays(n, src[keep], dst[keep]), new_of_old

def run(gr, sources, label):
    with Engine(gr) as e:
        e.set_option("groups", 32)
        e.run(sources)
        best = 1e9
        for _ in range(3):
            bc, st = e.run(sources)
            best = min(best, st["ms_total"])
    print("%-28s %.2f ms  level %.2f ms" % (label, best, st["ms_level"]), flush=True)
    return bc

bc0 = run(g, srcs, "as generated")
t0 = time.perf_counter()
order = np.argsort(-deg, kind="stable")
g1, new_of_old = relabel(g, order)
print("relabel host time %.2f s" % (time.perf_counter() - t0))
bc1 = run(g1, sorted(new_of_old[srcs].tolist()), "degree-descending ids")
print("BC max rel diff", float(np.max(np.abs(bc1[new_of_old] - bc0) / np.maximum(np.abs(bc0), 1e-9))))
rng = np.random.default_rng(3)
order = rng.permutation(n)
g2, new2 = relabel(g, order)
run(g2, sorted(new2[srcs].tolist()), "random ids")

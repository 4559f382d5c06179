"""Dev tool (CPU): shape of the BFS levels of one group of 32 sources on a bench workload -- which side of a
level holds the arcs (the numbers behind the child-driven backward levels).

    python tools/level_shape.py [workload]

Per level: vertices sitting there in any lane, (vertex, lane) pairs, the arcs of those vertices (what a
parent-driven pull scans; what the children scan one level up) and the (DAG arc, lane) pairs to the next level.
Uses the oracle (test infrastructure) for the BFS; not part of the product path.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_2008_05718_b200 import generators as G
import bench
g, label = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "rmat20")
n = g.num_vertices
deg = np.diff(g.offsets)
src = bench.pick_sources(n, 1024)
src = [s for s in src if deg[s] > 0][:32]
t=time.time()
D = np.stack([np.asarray(O.brandes_single_source(g, s)[0]) for s in src])
print("bfs", time.time()-t, D.shape, D.dtype)
col = g.col_idx; off = g.offsets
src_of_arc = np.repeat(np.arange(n), deg)
maxL = int(D[D < 10**6].max())
A = len(col)
print("arcs", A)
for L in range(0, maxL + 1):
    atL = (D == L)
    anyL = atL.any(axis=0)
    pairs = int(atL.sum())
    scan = int(deg[anyL].sum())
    hits = 0
    if L < maxL:
        for l in range(len(src)):
            hits += int(((D[l, src_of_arc] == L) & (D[l, col] == L + 1)).sum())
    print(f"L={L} verts_any={int(anyL.sum())} pairs={pairs} scan_arcs={scan} ({scan/A:.3f} of arcs) dag_arcs_to_next={hits}")

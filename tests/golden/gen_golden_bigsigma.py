"""Golden vectors in the regime where path counts exceed 2^53 (SURVEY.md hard part 1).

Run in the build container only (imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden_bigsigma.py

A full 40 x 32 lattice has ~70 BFS levels from a corner and its path counts grow about one bit
per level.  The reference's sequential Brandes oracle (oracle.py:29-67) carries them as exact
Python integers; this script records, for a few sources, its distances, its path counts
(correctly rounded to fp64 with ``float(int)``, plus log2 of the largest one and the exact
decimal digits of the largest one per source) and its fp64 dependencies, and the BC vector over
those sources (oracle.py:70-82).  The committed ``bigsigma_vectors.npz`` is what the C oracle port
and the GPU engine are compared with above 2^53: path counts at 1e-12 relative, delta / BC at 1e-9.
"""
import math
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

import hybir as H  # noqa: E402
from hybir.oracle import brandes_bc, brandes_single_source  # noqa: E402

from paper_2008_05718_b200 import generators as G  # noqa: E402

ROWS, COLS = 40, 32
g = G.grid(ROWS, COLS)
und = g.arc_src < g.arc_dst
rg = H.from_edges(g.num_vertices, [(int(u), int(v), 1) for u, v in zip(g.arc_src[und], g.arc_dst[und])])
sources = [0, COLS - 1, (ROWS // 2) * COLS + COLS // 2, ROWS * COLS - 1, 7 * COLS + 3]
dist = np.zeros((len(sources), g.num_vertices), dtype=np.int32)
sigma = np.zeros((len(sources), g.num_vertices), dtype=np.float64)
delta = np.zeros((len(sources), g.num_vertices), dtype=np.float64)
top_digits, top_log2 = [], []
for i, s in enumerate(sources):
    d, sg, dl = brandes_single_source(rg, s)
    dist[i] = [-1 if x is None else x for x in d]
    sigma[i] = [float(x) for x in sg]             # exact int -> nearest fp64
    delta[i] = dl
    big = max(sg)
    top_digits.append(str(big))
    top_log2.append(math.log2(big))
bc = brandes_bc(rg, sources).bc
assert max(top_log2) > 53, "the graph must leave the exact-integer range of fp64"
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bigsigma_vectors.npz")
np.savez_compressed(out, rows=ROWS, cols=COLS, sources=np.asarray(sources), dist=dist, sigma=sigma, delta=delta,
                    bc=np.asarray(bc, dtype=np.float64), sigma_max_log2=np.asarray(top_log2),
                    sigma_max_digits=np.asarray(top_digits))
print("wrote", out, os.path.getsize(out), "bytes; log2(max sigma) per source:", [round(x, 1) for x in top_log2])

"""Seeded synthetic graphs for the BASELINE.json configurations.

Definitions follow SURVEY.md section 8(d): R-MAT with (a,b,c,d) =
(0.57,0.19,0.19,0.05) drawn bit by bit from ``numpy.random.default_rng(seed)``
with no vertex permutation; 4-neighbour grids built like the reference test
factory (reference pkg/tests/conftest.py:36-47); a road-like thinning of the
grid (random spanning tree + a fraction of the remaining grid edges); and
Erdos-Renyi as uniform random endpoint pairs.  All of them go through
``from_edge_arrays`` so they carry the reference's normalisation.
"""

from __future__ import annotations

import numpy as np

from .graph import Graph, from_edge_arrays

__all__ = ["rmat", "rmat_edges", "grid", "road_like", "erdos_renyi", "path", "random_connected"]


def rmat_edges(scale: int, edge_factor: int, seed: int = 1, a=0.57, b=0.19, c=0.19):
    """Raw R-MAT endpoint draws (before normalisation)."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = n * edge_factor
    if scale > 31:
        raise ValueError("R-MAT scale above 31 is not supported")
    # endpoint bits are collected in 32-bit words (half the memory traffic of int64)
    u = np.zeros(m, dtype=np.uint32)
    v = np.zeros(m, dtype=np.uint32)
    r = np.empty(m, dtype=np.float64)
    for bit in range(scale):
        rng.random(m, out=r)                       # (same stream as rng.random(m))
        ub = r >= a + b
        vb = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u |= ub.astype(np.uint32) << np.uint32(bit)
        v |= vb.astype(np.uint32) << np.uint32(bit)
    u, v = u.astype(np.int64), v.astype(np.int64)
    return n, u, v


def rmat(scale: int, edge_factor: int, seed: int = 1, a=0.57, b=0.19, c=0.19) -> Graph:
    n, u, v = rmat_edges(scale, edge_factor, seed, a, b, c)
    return from_edge_arrays(n, u, v)


def _grid_edges(rows: int, cols: int):
    vid = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    hu, hv = vid[:, :-1].ravel(), vid[:, 1:].ravel()
    vu, vv = vid[:-1, :].ravel(), vid[1:, :].ravel()
    return np.concatenate([hu, vu]), np.concatenate([hv, vv])


def grid(rows: int, cols: int) -> Graph:
    u, v = _grid_edges(rows, cols)
    return from_edge_arrays(rows * cols, u, v)


def road_like(rows: int, cols: int, keep: float = 0.2, seed: int = 1) -> Graph:
    """Random spanning tree of the grid plus ``keep`` of the other grid edges.

    The tree is the minimum spanning tree under i.i.d. random edge ranks
    (= Kruskal over a random edge order), which keeps the diameter high and
    the path counts far below a full lattice (hard
    part 1).
    """
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import minimum_spanning_tree

    rng = np.random.default_rng(seed)
    u, v = _grid_edges(rows, cols)
    n = rows * cols
    rank = rng.permutation(len(u)).astype(np.float64) + 1.0
    mst = minimum_spanning_tree(coo_matrix((rank, (u, v)), shape=(n, n)).tocsr()).tocoo()
    # Map tree edges back to edge positions through their (unique) rank.
    by_rank = np.empty(len(u) + 1, dtype=np.int64)
    by_rank[rank.astype(np.int64)] = np.arange(len(u))
    in_tree = np.zeros(len(u), dtype=bool)
    in_tree[by_rank[np.rint(mst.data).astype(np.int64)]] = True
    extra = (~in_tree) & (rng.random(len(u)) < keep)
    sel = in_tree | extra
    return from_edge_arrays(n, u[sel], v[sel])


def erdos_renyi(n: int, num_pairs: int, seed: int = 1) -> Graph:
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, size=num_pairs, dtype=np.int64)
    v = rng.integers(0, n, size=num_pairs, dtype=np.int64)
    return from_edge_arrays(n, u, v)


def path(n: int) -> Graph:
    a = np.arange(n - 1, dtype=np.int64)
    return from_edge_arrays(n, a, a + 1)


def random_connected(n: int, extra_edges: int = 0, seed: int = 0, weighted: bool = False) -> Graph:
    """Random spanning tree + extra edges, always connected; unit weights, or
    integer weights 1..10 with ``weighted=True``.

    Same construction and the same ``random.Random(seed)`` draw order as the
    reference test factory (conftest.py:10-29), so a given
    (n, extra_edges, weighted, seed) is the same graph on both sides.
    """
    import random

    rng = random.Random(seed)
    nodes = list(range(n))
    rng.shuffle(nodes)
    us, vs, ws = [], [], []
    for i in range(1, n):
        us.append(nodes[rng.randrange(i)])
        vs.append(nodes[i])
        if weighted:
            ws.append(rng.randint(1, 10))
    added = 0
    while added < extra_edges:
        a, b = rng.randrange(n), rng.randrange(n)
        if a == b:
            continue
        us.append(a), vs.append(b)
        if weighted:
            ws.append(rng.randint(1, 10))
        added += 1
    return from_edge_arrays(n, us, vs, ws if weighted else None)

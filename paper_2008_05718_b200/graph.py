"""Host-side graph container: normalised undirected graph in CSR form.

Mirrors the reference ``Graph`` / ``from_edges`` contract
(reference pkg/src/hybir/graph.py:21-110): every undirected edge is stored as
two directed arcs, arcs are sorted by (src, dst), self loops are dropped,
parallel edges collapse to the minimum weight, weights must be positive.

What is different, on purpose:

* construction is vectorised numpy (the reference walks a Python dict,
  graph.py:70-95, unusable beyond ~1e6 edges);
* the primary storage is what the GPU consumes -- ``offsets`` int64[n+1] and
  ``col_idx`` int32[2m]; the reference's ``arc_src`` / ``arc_dst`` /
  ``arc_weight`` / ``rev_arc`` int64 views are materialised lazily so an
  R-MAT scale-24 graph does not pay 16 GB of host memory for arrays the
  unit-weight GPU path never reads.
"""

from __future__ import annotations

import hashlib

import numpy as np

from .errors import DomainError, FormatError, ParseError

__all__ = [
    "Graph",
    "from_edges",
    "from_edge_arrays",
    "load_edge_list",
    "load_dimacs_gr",
    "write_edge_list",
    "graph_stats",
    "as_graph",
]


class Graph:
    """Immutable normalised graph (shared read-only, reference SPEC.md:73)."""

    def __init__(self, num_vertices, num_edges, offsets, col_idx, weights=None):
        self.num_vertices = int(num_vertices)
        self.num_edges = int(num_edges)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        # None means "all ones" (the only case the GPU path accepts).
        self._weights = None if weights is None else np.ascontiguousarray(weights, dtype=np.int64)
        self._cache = {}

    # -- reference-compatible views (graph.py:21-61) ----------------------
    @property
    def num_arcs(self) -> int:
        # = 2 * num_edges for a normalised graph; a rank-local view (rows of one part only,
        # partitioned.py) holds every cut arc once, so count what is stored
        return int(len(self.col_idx))

    @property
    def unit_weight(self) -> bool:
        return self._weights is None

    @property
    def arc_dst(self) -> np.ndarray:
        if "dst" not in self._cache:
            self._cache["dst"] = self.col_idx.astype(np.int64)
        return self._cache["dst"]

    @property
    def arc_src(self) -> np.ndarray:
        if "src" not in self._cache:
            deg = np.diff(self.offsets)
            self._cache["src"] = np.repeat(np.arange(self.num_vertices, dtype=np.int64), deg)
        return self._cache["src"]

    @property
    def arc_weight(self) -> np.ndarray:
        if self._weights is not None:
            return self._weights
        if "wt" not in self._cache:
            self._cache["wt"] = np.ones(self.num_arcs, dtype=np.int64)
        return self._cache["wt"]

    @property
    def rev_arc(self) -> np.ndarray:
        # Position of arc (v,u) for every arc (u,v); arcs are unique and
        # sorted by (src,dst) so a binary search on the packed key finds it.
        if "rev" not in self._cache:
            n = max(self.num_vertices, 1)
            keys = self.arc_src * n + self.arc_dst
            self._cache["rev"] = np.searchsorted(keys, self.arc_dst * n + self.arc_src)
        return self._cache["rev"]

    @property
    def inf_distance(self) -> int:
        """Sentinel above every achievable distance (graph.py:34-38)."""
        if self._weights is None:
            return self.num_edges + 1
        return int(self._weights.sum()) // 2 + 1

    @property
    def adjacency(self):
        """Plain-list copies (graph.py:40-48); only sensible for small graphs."""
        if "adj" not in self._cache:
            self._cache["adj"] = (
                self.offsets.tolist(),
                self.arc_dst.tolist(),
                self.arc_weight.tolist(),
                self.rev_arc.tolist(),
            )
        return self._cache["adj"]

    def pin(self) -> "Graph":
        """Move ``offsets`` / ``col_idx`` into page-locked host memory so the
        host-to-device copy of the CSR runs at full PCIe speed (no-op without
        CUDA).  torch is used only as the pinned allocator."""
        if self._cache.get("pinned"):
            return self
        try:
            import torch
            if not torch.cuda.is_available():
                return self
            for name in ("offsets", "col_idx"):
                arr = getattr(self, name)
                t = torch.empty(arr.shape, dtype=torch.int64 if arr.dtype == np.int64 else torch.int32,
                                pin_memory=True)
                buf = t.numpy()
                buf[...] = arr
                self._cache["pin_" + name] = t      # keeps the allocation alive
                setattr(self, name, buf)
            self._cache["pinned"] = True
        except Exception:
            pass
        return self

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def arcs_of(self, v: int) -> range:
        return range(int(self.offsets[v]), int(self.offsets[v + 1]))

    def content_hash(self) -> str:
        h = hashlib.sha256()
        h.update(np.int64(self.num_vertices).tobytes())
        h.update(self.offsets.tobytes())
        h.update(self.col_idx.tobytes())
        if self._weights is not None:
            h.update(self._weights.tobytes())
        return h.hexdigest()

    def __repr__(self):
        return "Graph(n=%d, m=%d%s)" % (
            self.num_vertices, self.num_edges, "" if self.unit_weight else ", weighted")


def _first_bad(mask):
    idx = np.flatnonzero(mask)
    return int(idx[0]) if len(idx) else None


def from_edge_arrays(num_vertices: int, u, v, w=None) -> Graph:
    """Vectorised ``from_edges`` over endpoint arrays (graph.py:64-110 semantics)."""
    n = int(num_vertices)
    u = np.asarray(u, dtype=np.int64).ravel()
    v = np.asarray(v, dtype=np.int64).ravel()
    if u.shape != v.shape:
        raise FormatError("endpoint arrays differ in length")
    if w is not None:
        w = np.asarray(w, dtype=np.int64).ravel()
        if w.shape != u.shape:
            raise FormatError("weight array length differs from endpoint arrays")

    # The reference validates edge by edge and raises on the first offender
    # (range first, then negative, then zero weight); keep that precedence.
    bad_range = (u < 0) | (u >= n) | (v < 0) | (v >= n)
    first = [(_first_bad(bad_range), 0)]
    if w is not None:
        first.append((_first_bad(w < 0), 1))
        first.append((_first_bad(w == 0), 2))
    first = [(i, kind) for i, kind in first if i is not None]
    if first:
        i, kind = min(first)
        if kind == 0:
            raise FormatError("vertex out of range: (%d, %d), n=%d" % (u[i], v[i], n))
        if kind == 1:
            raise DomainError("negative weight %d on edge (%d, %d)" % (w[i], u[i], v[i]))
        raise DomainError(
            "zero weight on edge (%d, %d); distance levels must be strict" % (u[i], v[i]))

    keep = u != v
    lo = np.minimum(u, v)[keep]
    hi = np.maximum(u, v)[keep]
    key = lo * max(n, 1) + hi
    if w is None:
        # sort + neighbour compare (np.unique on 10^8 keys is two orders of magnitude slower)
        key = np.sort(key)
        if len(key):
            firsts = np.ones(len(key), dtype=bool)
            np.not_equal(key[1:], key[:-1], out=firsts[1:])
            key = key[firsts]
        wk = None
    else:
        wk = w[keep]
        order = np.lexsort((wk, key))
        key, wk = key[order], wk[order]
        firsts = np.ones(len(key), dtype=bool)
        firsts[1:] = key[1:] != key[:-1]
        key, wk = key[firsts], wk[firsts]
        if len(wk) == 0 or bool((wk == 1).all()):
            wk = None
    m = len(key)
    lo = key // max(n, 1)
    hi = key - lo * max(n, 1)

    nn = max(n, 1)
    offsets = np.zeros(n + 1, dtype=np.int64)
    if wk is None:
        # arcs are unique: sorting the packed (src, dst) keys is the whole job
        arcs = np.concatenate([key, hi * nn + lo])
        arcs.sort()
        src = arcs // nn
        dst_sorted = (arcs - src * nn).astype(np.int32)
        counts = np.bincount(src, minlength=n) if n else np.zeros(0, dtype=np.int64)
        np.cumsum(counts, out=offsets[1:])
        return Graph(n, m, offsets, dst_sorted, None)
    src = np.concatenate([lo, hi])
    dst = np.concatenate([hi, lo])
    order = np.argsort(src * nn + dst, kind="stable")
    dst_sorted = dst[order]
    counts = np.bincount(src, minlength=n) if n else np.zeros(0, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    weights = np.concatenate([wk, wk])[order]
    return Graph(n, m, offsets, dst_sorted.astype(np.int32), weights)


def from_edges(num_vertices: int, edges) -> Graph:
    """Build a normalised Graph from (u, v, w) triples or an (E, 2|3) array."""
    if isinstance(edges, np.ndarray):
        arr = edges
    else:
        edges = list(edges)
        if not edges:
            arr = np.zeros((0, 3), dtype=np.int64)
        else:
            arr = np.asarray(edges, dtype=np.int64)
    if arr.ndim != 2 or arr.shape[1] not in (2, 3):
        raise FormatError("edges must be (u, v, w) triples or an (E, 2|3) array")
    w = arr[:, 2] if arr.shape[1] == 3 else None
    return from_edge_arrays(num_vertices, arr[:, 0], arr[:, 1], w)


def load_edge_list(path, weighted: bool = False) -> Graph:
    """Read ``u v [w]`` lines; ``#`` / ``%`` start comments (graph.py:113-136)."""
    us, vs, ws = [], [], []
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line or line[0] in "#%":
                continue
            parts = line.split()
            if len(parts) not in (2, 3):
                raise ParseError("expected 'u v [w]', got %r" % line, lineno)
            try:
                a, b = int(parts[0]), int(parts[1])
                c = int(parts[2]) if (weighted and len(parts) == 3) else 1
            except ValueError:
                raise ParseError("non-integer field in %r" % line, lineno) from None
            if a < 0 or b < 0:
                raise ParseError("negative vertex id in %r" % line, lineno)
            if c < 0:
                raise DomainError("line %d: negative weight %d" % (lineno, c))
            us.append(a), vs.append(b), ws.append(c)
    n = (max(max(us), max(vs)) + 1) if us else 0
    return from_edge_arrays(n, us, vs, ws)


def load_dimacs_gr(path) -> Graph:
    """DIMACS shortest-path format (graph.py:139-173): ``c`` comments, one ``p sp n m`` problem
    line, then ``a u v w`` arcs with 1-based vertex ids; the arc count must match the header."""
    n = declared = None
    us, vs, ws = [], [], []
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            tok = raw.split()
            if not tok or tok[0].startswith("c"):
                continue
            if tok[0] == "p":
                if len(tok) != 4 or tok[1] != "sp":
                    raise ParseError("bad problem line %r" % raw.strip(), lineno)
                n, declared = int(tok[2]), int(tok[3])
            elif tok[0] == "a":
                if n is None:
                    raise ParseError("arc line before problem line", lineno)
                if len(tok) != 4:
                    raise ParseError("bad arc line %r" % raw.strip(), lineno)
                a, b, c = int(tok[1]), int(tok[2]), int(tok[3])
                if not (1 <= a <= n and 1 <= b <= n):
                    raise FormatError("line %d: vertex out of range in %r (n=%d)" % (lineno, raw.strip(), n))
                us.append(a - 1), vs.append(b - 1), ws.append(c)
            else:
                raise ParseError("unknown line type %r" % tok[0], lineno)
    if n is None:
        raise FormatError("missing problem line")
    if declared != len(us):
        raise FormatError("header declares %d arcs, file has %d" % (declared, len(us)))
    return from_edge_arrays(n, us, vs, ws)


def write_edge_list(g: Graph, path, weighted: bool = True) -> None:
    src, dst, wt = g.arc_src, g.arc_dst, g.arc_weight
    keep = src < dst
    with open(path, "w") as fh:
        for a, b, c in zip(src[keep].tolist(), dst[keep].tolist(), wt[keep].tolist()):
            fh.write("%d %d %d\n" % (a, b, c) if weighted else "%d %d\n" % (a, b))


def graph_stats(g: Graph) -> dict:
    n, m = g.num_vertices, g.num_edges
    if n == 0:
        return {"n": 0, "m": 0, "avg_degree": 0.0, "max_degree": 0}
    deg = np.diff(g.offsets)
    return {"n": n, "m": m, "avg_degree": 2.0 * m / n, "max_degree": int(deg.max())}


def as_graph(X) -> Graph:
    """Coerce a Graph, a path, or an (E, 2|3) edge array (graph.py:200-216)."""
    if isinstance(X, Graph):
        return X
    if isinstance(X, (str, bytes)) or hasattr(X, "__fspath__"):
        return load_edge_list(X)
    arr = np.asarray(X)
    if arr.ndim != 2 or arr.shape[1] not in (2, 3):
        raise FormatError("expected a Graph, a path, or an (n_edges, 2|3) array of edges")
    n = int(arr[:, :2].max()) + 1 if len(arr) else 0
    return from_edges(n, arr.astype(np.int64))

"""Generate tests/golden/reference_vectors_weighted.json by running the REFERENCE package
on weighted graphs (positive integer weights; the reference's Dijkstra paths).

Run in the build container only (it imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden_weighted.py

Graphs: the reference's weighted-tie fixture ``w5`` (conftest.py:77-81), the weighted members of
its acceptance-corpus family (``random_connected_graph(n, extra, weighted=True, seed)``,
conftest.py:10-29, test_acceptance.py:69-153) and two weighted grids.  Recorded per graph: the
sequential Brandes oracle per source (oracle.py:29-82), the partition, and ``run_bc`` in both
modes with its per-source reports (engine.py:120-153).
"""

import json
import os
import random
import sys
import tempfile

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import hybir as H  # noqa: E402
from hybir.engine import RunConfig, run_bc  # noqa: E402
from hybir.oracle import brandes_bc, brandes_single_source  # noqa: E402


def corpus_edges(n, extra_edges, seed):
    """conftest.py:10-29 with weighted=True, as (u, v, w) triples."""
    rng = random.Random(seed)
    nodes = list(range(n))
    rng.shuffle(nodes)
    edges = []
    for i in range(1, n):
        u = nodes[rng.randrange(i)]
        v = nodes[i]
        edges.append((u, v, rng.randint(1, 10)))
    added = 0
    while added < extra_edges:
        u, v = rng.randrange(n), rng.randrange(n)
        if u == v:
            continue
        edges.append((u, v, rng.randint(1, 10)))
        added += 1
    return edges


def grid_edges(rows, cols, seed, wmax):
    rng = random.Random(seed)
    edges = []
    for r in range(rows):
        for c in range(cols):
            if c + 1 < cols:
                edges.append((r * cols + c, r * cols + c + 1, rng.randint(1, wmax)))
            if r + 1 < rows:
                edges.append((r * cols + c, (r + 1) * cols + c, rng.randint(1, wmax)))
    return edges


def graphs():
    out = [("w5", 5, [(0, 1, 2), (0, 2, 1), (1, 2, 1), (1, 3, 3), (2, 3, 4), (3, 4, 1)], "half")]
    for n, extra, seed, ratio in ((12, 6, 1001, 0.5), (25, 25, 1003, 0.7), (40, 50, 1005, 0.5),
                                  (70, 100, 1007, 0.5), (120, 200, 1009, 0.7)):
        out.append(("wrc_n%d_s%d" % (n, seed), n, corpus_edges(n, extra, seed), ("greedy", ratio, seed)))
    out.append(("wgrid7x6", 42, grid_edges(7, 6, 5, 3), "half"))
    out.append(("wgrid10x9_w2", 90, grid_edges(10, 9, 6, 2), ("greedy", 0.5, 2)))
    return out


def main():
    doc = {"generator": "tests/golden/gen_golden_weighted.py", "reference": "hybir 0.1.0", "graphs": []}
    for name, n, edges, part in graphs():
        g = H.from_edges(n, edges)
        if part == "half":
            a = np.zeros(n, dtype=np.int8)
            a[n // 2:] = 1
            p = H.Partition(a, 0.5)
        else:
            _, ratio, seed = part
            p = H.greedy_bipartition(g, ratio, seed=seed)
        bs = H.identify_borders(g, p)
        rng = random.Random(7)
        srcs = list(range(n)) if n <= 30 else sorted(rng.sample(range(n), 12))
        rec = {
            "name": name, "n": n, "inf": int(g.inf_distance),
            "edges": [[int(u), int(v), int(w)] for u, v, w in zip(g.arc_src, g.arc_dst, g.arc_weight) if u < v],
            "assignment": [int(x) for x in p.assignment],
            "borders": [list(map(int, b)) for b in bs.borders],
            "bc_all_sources": brandes_bc(g).bc.tolist(),
            "sources": [],
        }
        for s in srcs:
            dist, sigma, delta = brandes_single_source(g, s)
            rec["sources"].append({"s": s, "dist": [-1 if d is None else int(d) for d in dist],
                                   "sigma": [int(x) for x in sigma], "delta": [float(x) for x in delta]})
        with tempfile.NamedTemporaryFile("w", suffix=".part", delete=False) as fh:
            fh.write("\n".join(str(int(x)) for x in p.assignment) + "\n")
            pfile = fh.name
        for mode in ("hybir", "bsp-baseline"):
            res = run_bc(g, RunConfig(sources=srcs, mode=mode, partition_file=pfile))
            key = mode.replace("-", "_")
            rec["run_bc_" + key] = res.bc.tolist()
            rec["per_source_" + key] = res.per_source
        os.unlink(pfile)
        rec["run_bc_sources"] = srcs
        doc["graphs"].append(rec)
        print(name, "n=%d m=%d borders=%s max dist=%d" % (
            n, g.num_edges, bs.counts(), max(max(x for x in sr["dist"]) for sr in rec["sources"])))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors_weighted.json")
    with open(path, "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

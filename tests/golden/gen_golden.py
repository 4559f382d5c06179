"""Generate tests/golden/reference_vectors.json by running the REFERENCE package.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

For a fixed set of small unit-weight graphs it records what the reference's
own code computes on the BC hot path: the sequential Brandes oracle
(oracle.py:29-82), ``initial_relax`` (relax.py:42-103), the partition /
borders / border matrices (partition.py, border_matrix.py:48-67), the hybir
forward phase with its reports and border frontier (forward.py:188-256),
the backward phase reports (backward.py:59-151), the bsp-baseline reports
(bsp.py:22-142) and ``run_bc`` in both modes (engine.py:120-153).
The committed JSON is what the repo's tests compare against.
"""

import json
import os
import random
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

import hybir as H  # noqa: E402
from hybir.backward import backward_phase  # noqa: E402
from hybir.bsp import bsp_backward, bsp_forward  # noqa: E402
from hybir.engine import RunConfig, run_bc  # noqa: E402
from hybir.forward import forward_phase, merge_states  # noqa: E402
from hybir.oracle import brandes_bc, brandes_single_source  # noqa: E402
from hybir.relax import initial_relax  # noqa: E402

from paper_2008_05718_b200 import generators as G  # noqa: E402


def ref_graph(n, edges):
    return H.from_edges(n, [(u, v, 1) for u, v in edges])


def edges_of(g):
    return [[int(u), int(v)] for u, v in zip(g.arc_src, g.arc_dst) if u < v]


def half_split(n):
    a = np.zeros(n, dtype=np.int8)
    a[n // 2:] = 1
    return a


def graphs():
    out = []
    out.append(("p4", 4, [(i, i + 1) for i in range(3)], "half"))
    out.append(("diamond", 4, [(0, 1), (0, 2), (1, 3), (2, 3)], "half"))
    out.append(("c6", 6, [(i, (i + 1) % 6) for i in range(6)], "half"))
    out.append(("k4", 4, [(i, j) for i in range(4) for j in range(i + 1, 4)], "half"))
    out.append(("star5", 5, [(0, i) for i in range(1, 5)], "half"))
    out.append(("p64", 64, [(i, i + 1) for i in range(63)], "half"))
    out.append(("two_components", 6, [(0, 1), (1, 2), (3, 4), (4, 5)], "half"))
    out.append(("no_cut_reach", 5, [(0, 1), (2, 3), (3, 4)], [0, 0, 0, 1, 1]))
    gg = G.grid(6, 5)
    out.append(("grid6x5", 30, [tuple(e) for e in edges_of(gg)], "half"))
    gg = G.grid(9, 7)
    out.append(("grid9x7_greedy", 63, [tuple(e) for e in edges_of(gg)], ("greedy", 0.5, 3)))
    # the unweighted members of the reference's acceptance-corpus family
    # (random_connected_graph(n, extra, weighted=False, seed), conftest.py:10-29)
    for n, extra, seed, ratio in ((12, 5, 1000, 0.7), (25, 20, 1002, 0.5), (40, 60, 1004, 0.5),
                                  (60, 30, 1006, 0.7), (90, 90, 1008, 0.5)):
        gg = G.random_connected(n, extra, seed)
        out.append(("rc_n%d_s%d" % (n, seed), n, [tuple(e) for e in edges_of(gg)],
                    ("greedy", ratio, seed)))
    gg = G.rmat(8, 4, 1)
    out.append(("rmat8", 256, [tuple(e) for e in edges_of(gg)], ("greedy", 0.5, 0)))
    return out


def main():
    doc = {"generator": "tests/golden/gen_golden.py", "reference": "hybir 0.1.0", "graphs": []}
    for name, n, edges, part in graphs():
        g = ref_graph(n, edges)
        if part == "half":
            assignment = half_split(n)
            p = H.Partition(assignment, 0.5)
        elif isinstance(part, list):
            p = H.Partition(np.array(part, dtype=np.int8), 0.5)
        else:
            _, ratio, seed = part
            p = H.greedy_bipartition(g, ratio, seed=seed)
        bs = H.identify_borders(g, p)
        bmx = H.compute_border_matrices(g, p, bs)
        inf = g.inf_distance
        rng = random.Random(7)
        srcs = list(range(n)) if n <= 30 else sorted(rng.sample(range(n), 12))
        rec = {
            "name": name, "n": n, "edges": edges_of(g), "inf": int(inf),
            "offsets": g.offsets.tolist(), "arc_dst": g.arc_dst.tolist(),
            "assignment": [int(x) for x in p.assignment],
            "borders": [list(map(int, b)) for b in bs.borders],
            "cut_arcs": [[int(u), int(v)] for u, v, _ in bs.cut_arcs],
            "bm": [np.where(m >= inf, -1, m).tolist() for m in bmx.bm],
            "sm": [[[int(x) for x in row] for row in side] for side in bmx.sm],
            "bc_all_sources": brandes_bc(g).bc.tolist(),
            "sources": [],
        }
        for s in srcs:
            dist, sigma, delta = brandes_single_source(g, s)
            states, frep, bf = forward_phase(g, p, bs, bmx, s)
            hdist, hsigma, _ = merge_states(g, p, states)
            hdelta, brep = backward_phase(g, p, bs, states, s)
            bstates, bsp_f = bsp_forward(g, p, s)
            _, bsp_b = bsp_backward(g, p, bs, bstates, s)
            sp = int(p.assignment[s])
            step1 = initial_relax(g, p.mask(sp), [(s, 0, 1)])
            rec["sources"].append({
                "s": s,
                "dist": [-1 if d is None else int(d) for d in dist],
                "sigma": [int(x) for x in sigma],
                "delta": [float(x) for x in delta],
                "hybir_dist": [-1 if d >= inf else int(d) for d in hdist],
                "hybir_sigma": [int(x) for x in hsigma],
                "hybir_delta": [float(x) for x in hdelta],
                "step1_dist": [-1 if d >= inf else int(d) for d in step1.dist],
                "step1_sigma": [int(x) for x in step1.sigma],
                "forward": frep.as_dict(),
                "backward": brep.as_dict(),
                "border_dist": [[-1 if d >= inf else int(d) for d in side] for side in bf.dist],
                "border_sigma": [[int(x) for x in side] for side in bf.sigma],
                "arrival_sigma": [[int(x) for x in side] for side in bf.arrival_sigma],
                "bsp_forward": bsp_f,
                "bsp_backward": bsp_b,
            })
        # run_bc through the reference engine, explicit partition via a temp file
        import tempfile
        with tempfile.NamedTemporaryFile("w", suffix=".part", delete=False) as fh:
            fh.write("\n".join(str(int(x)) for x in p.assignment) + "\n")
            pfile = fh.name
        for mode in ("hybir", "bsp-baseline"):
            res = run_bc(g, RunConfig(sources=srcs, mode=mode, partition_file=pfile))
            rec["run_bc_" + mode.replace("-", "_")] = res.bc.tolist()
        os.unlink(pfile)
        rec["run_bc_sources"] = srcs
        doc["graphs"].append(rec)
        print(name, "n=%d m=%d borders=%s" % (n, g.num_edges, bs.counts()))
    # seeded multi-seed relax cases (relax.py:42-103): staggered seeds and masks
    relax_cases = []
    rng = random.Random(11)
    for case in range(12):
        n = rng.randint(8, 40)
        gg = G.random_connected(n, rng.randint(0, n), seed=200 + case)
        g = ref_graph(n, [tuple(e) for e in edges_of(gg)])
        mask = [rng.random() < 0.75 for _ in range(n)]
        inside = [v for v in range(n) if mask[v]]
        seeds = [(rng.choice(inside), rng.randint(0, 5), rng.randint(0, 3)) for _ in range(rng.randint(1, 6))]
        res = initial_relax(g, mask, seeds)
        relax_cases.append({
            "n": n, "edges": edges_of(g), "mask": [int(x) for x in mask],
            "seeds": [list(map(int, x)) for x in seeds],
            "dist": [-1 if d >= g.inf_distance else int(d) for d in res.dist],
            "sigma": [int(x) for x in res.sigma],
        })
    doc["relax_cases"] = relax_cases
    # config-1 anchor: R-MAT scale-12 EF-8 (the reference-runnable BASELINE config)
    g12 = G.rmat(12, 8, 1)
    rg = H.Graph(g12.num_vertices, g12.num_edges, g12.offsets, g12.arc_src, g12.arc_dst,
                 g12.arc_weight, g12.rev_arc)
    anchor = {"n": g12.num_vertices, "m": g12.num_edges, "sources": []}
    for s in (0, 1, 17, 999, 2048, 4000):
        dist, sigma, delta = brandes_single_source(rg, s)
        d = np.array([-1 if x is None else x for x in dist])
        anchor["sources"].append({
            "s": s, "reached": int((d >= 0).sum()), "ecc": int(d.max()),
            "sigma_sum": int(sum(sigma)), "sigma_max": int(max(sigma)),
            "delta_sum": float(np.sum(delta)), "delta_max": float(np.max(delta)),
            "dist_hist": np.bincount(d[d >= 0]).tolist(),
        })
    doc["rmat12_anchor"] = anchor
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")
    with open(path, "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

"""Pins the CPU oracle (oracle/) to the reference: known-answer vectors the
reference's own tests hold and golden vectors produced
by running the reference package (tests/golden/gen_golden.py)."""

import numpy as np
import pytest

import oracle as O
from paper_2008_05718_b200 import from_edges, generators as G

from conftest import graph_from_record


def _named(name):
    if name == "p4":
        return G.path(4)
    if name == "diamond":
        return from_edges(4, [(0, 1, 1), (0, 2, 1), (1, 3, 1), (2, 3, 1)])
    if name == "c6":
        return from_edges(6, [(i, (i + 1) % 6, 1) for i in range(6)])
    if name == "k4":
        return from_edges(4, [(i, j, 1) for i in range(4) for j in range(i + 1, 4)])
    if name == "star5":
        return from_edges(5, [(0, i, 1) for i in range(1, 5)])
    raise KeyError(name)


# reference pkg/tests/test_oracle.py:37-42
@pytest.mark.parametrize("name,expect", [
    ("p4", [0, 4, 4, 0]), ("diamond", [1, 1, 1, 1]), ("c6", [4] * 6), ("k4", [0] * 4),
    ("star5", [12, 0, 0, 0, 0]),
])
def test_known_bc(name, expect):
    bc, _ = O.brandes_bc(_named(name))
    assert np.allclose(bc, expect, rtol=1e-12, atol=1e-12)


def test_known_single_source_vectors():
    # reference pkg/tests/test_backward.py:25-37
    d, s, dl, _ = O.brandes_single_source(_named("p4"), 0)
    assert d.tolist() == [0, 1, 2, 3] and s.tolist() == [1, 1, 1, 1] and dl.tolist() == [3, 2, 1, 0]
    d, s, dl, _ = O.brandes_single_source(_named("diamond"), 0)
    assert d.tolist() == [0, 1, 1, 2] and s.tolist() == [1, 1, 1, 2] and dl.tolist() == [3, 0.5, 0.5, 0]
    d, s, dl, _ = O.brandes_single_source(_named("star5"), 1)
    assert dl[0] == 3.0
    # reference pkg/tests/test_forward.py:151-156
    d, s, _, _ = O.brandes_single_source(_named("c6"), 0)
    assert d.tolist() == [0, 1, 2, 3, 2, 1] and s.tolist() == [1, 1, 1, 2, 1, 1]


def test_known_relax_vectors():
    p4 = _named("p4")
    # reference pkg/tests/test_forward.py:18-41
    d, s = O.masked_relax(p4, None, [(0, 0, 1)])
    assert d.tolist() == [0, 1, 2, 3] and s.tolist() == [1, 1, 1, 1]
    d, s = O.masked_relax(p4, [1, 1, 0, 0], [(0, 0, 1)])
    assert d.tolist() == [0, 1, p4.inf_distance, p4.inf_distance] and s[2] == 0
    d, s = O.masked_relax(p4, None, [(0, 0, 2), (3, 0, 3)])
    assert d.tolist() == [0, 1, 1, 0] and s.tolist() == [2, 2, 3, 3]
    d, s = O.masked_relax(p4, None, [(0, p4.inf_distance, 1), (1, 0, 0)])
    assert (d == p4.inf_distance).all()
    with pytest.raises(LookupError):
        O.masked_relax(p4, [1, 1, 0, 0], [(3, 0, 1)])
    d, s = O.masked_relax(_named("diamond"), None, [(0, 0, 1)])
    assert s.tolist() == [1, 1, 1, 2]


def test_single_source_matches_reference_vectors(golden_graphs):
    checked = 0
    for g, rec in golden_graphs.values():
        for src in rec["sources"]:
            d, s, dl, info = O.brandes_single_source(g, src["s"])
            assert d.tolist() == src["dist"]
            assert s.tolist() == [float(x) for x in src["sigma"]]
            assert info["sigma_max"] < 2.0 ** 53
            # same settle order and the same division -> bit-identical delta
            assert dl.tolist() == src["delta"]
            checked += 1
    assert checked > 150


def test_bc_matches_reference_vectors(golden_graphs):
    for g, rec in golden_graphs.values():
        for threads in (1, 3):
            bc, _ = O.brandes_bc(g, threads=threads)
            assert np.allclose(bc, rec["bc_all_sources"], rtol=1e-12, atol=1e-12)
        bc, _ = O.brandes_bc(g, rec["run_bc_sources"], threads=2)
        assert np.allclose(bc, rec["run_bc_hybir"], rtol=1e-9, atol=1e-12)
        assert np.allclose(bc, rec["run_bc_bsp_baseline"], rtol=1e-9, atol=1e-12)


def test_masked_relax_matches_reference_vectors(golden):
    for case in golden["relax_cases"]:
        g = graph_from_record(case)
        d, s = O.masked_relax(g, case["mask"], [tuple(x) for x in case["seeds"]])
        d = np.where(d >= g.inf_distance, -1, d)
        assert d.tolist() == case["dist"]
        assert s.tolist() == [float(x) for x in case["sigma"]]


def test_step1_relax_matches_reference_vectors(golden_graphs):
    for g, rec in golden_graphs.values():
        a = np.asarray(rec["assignment"])
        for src in rec["sources"][:6]:
            s = src["s"]
            d, sg = O.masked_relax(g, a == a[s], [(s, 0, 1)])
            d = np.where(d >= g.inf_distance, -1, d)
            assert d.tolist() == src["step1_dist"]
            assert sg.tolist() == [float(x) for x in src["step1_sigma"]]


def test_rmat12_anchor(golden, rmat12):
    # BASELINE config 1: the graph itself and six sources of the reference oracle
    anchor = golden["rmat12_anchor"]
    assert (rmat12.num_vertices, rmat12.num_edges) == (anchor["n"], anchor["m"]) == (4096, 26603)
    for rec in anchor["sources"]:
        d, s, dl, info = O.brandes_single_source(rmat12, rec["s"])
        assert info["reached"] == rec["reached"] and int(d.max()) == rec["ecc"]
        assert int(s.sum()) == rec["sigma_sum"] and int(s.max()) == rec["sigma_max"]
        assert np.bincount(d[d >= 0]).tolist() == rec["dist_hist"]
        assert float(dl.sum()) == pytest.approx(rec["delta_sum"], rel=1e-12)
        assert float(dl.max()) == pytest.approx(rec["delta_max"], rel=1e-12)


def test_counters_are_consistent(rmat12):
    d, s, dl, info = O.brandes_single_source(rmat12, 17)
    deg = np.diff(rmat12.offsets)
    assert info["arcs_reached"] == int(deg[d >= 0].sum())
    src, dst = rmat12.arc_src, rmat12.arc_dst
    tight = (d[src] >= 0) & (d[dst] == d[src] + 1)
    assert info["dag_arcs"] == int(tight.sum())


# ---- weighted graphs: the reference's heap Dijkstra (oracle.py:44-61) ------------------

def _weighted_golden():
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors_weighted.json")
    with open(path) as fh:
        return json.load(fh)


def weighted_graph_from_record(rec):
    return from_edges(rec["n"], [tuple(e) for e in rec["edges"]])


def test_weighted_tie_fixture_w5():
    # reference pkg/tests/test_oracle.py:31-34
    g = from_edges(5, [(0, 1, 2), (0, 2, 1), (1, 2, 1), (1, 3, 3), (2, 3, 4), (3, 4, 1)])
    assert not g.unit_weight
    d, s, _, _ = O.brandes_single_source(g, 0)
    assert d.tolist() == [0, 2, 1, 5, 6]
    assert s.tolist() == [1, 2, 1, 3, 3]


def test_weighted_oracle_matches_reference_golden():
    doc = _weighted_golden()
    assert len(doc["graphs"]) >= 8
    for rec in doc["graphs"]:
        g = weighted_graph_from_record(rec)
        assert g.inf_distance == rec["inf"]
        bc, _ = O.brandes_bc(g)
        assert np.allclose(bc, rec["bc_all_sources"], rtol=1e-12, atol=1e-12), rec["name"]
        for sr in rec["sources"]:
            d, s, dl, info = O.brandes_single_source(g, sr["s"])
            assert d.tolist() == sr["dist"], rec["name"]
            assert s.tolist() == sr["sigma"], rec["name"]
            assert np.array_equal(dl, np.array(sr["delta"])), rec["name"]     # same settle order: bit-identical
        bc_s, _ = O.brandes_bc(g, rec["run_bc_sources"], threads=1)
        assert np.allclose(bc_s, rec["run_bc_hybir"], rtol=1e-9, atol=1e-12)
        assert np.allclose(bc_s, rec["run_bc_bsp_baseline"], rtol=1e-9, atol=1e-12)


def test_path_counts_beyond_2_53_match_the_bigint_reference():
    """Above 2^53 the reference oracle keeps exact Python integers (oracle.py:56-61); the C port
    carries fp64.  Golden vectors from the reference itself on a 40 x 32 lattice (max sigma 2^66,
    tests/golden/gen_golden_bigsigma.py): distances exact, path counts within 1e-12 of the
    correctly rounded integers, dependencies / BC within 1e-9."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bigsigma_vectors.npz"))
    g = G.grid(int(z["rows"]), int(z["cols"]))
    srcs = z["sources"].tolist()
    assert z["sigma_max_log2"].max() > 53
    for i, s in enumerate(srcs):
        d, sg, dl, info = O.brandes_single_source(g, s)
        assert np.array_equal(d, z["dist"][i])
        assert np.allclose(sg, z["sigma"][i], rtol=1e-12, atol=0)
        assert np.allclose(dl, z["delta"][i], rtol=1e-9, atol=1e-12)
        # the recorded maximum really is the exact integer the reference computed
        assert float(int(str(z["sigma_max_digits"][i]))) == z["sigma"][i].max() == info["sigma_max"] or \
            abs(info["sigma_max"] / z["sigma"][i].max() - 1) < 1e-12
    bc, _ = O.brandes_bc(g, srcs)
    assert np.allclose(bc, z["bc"], rtol=1e-9, atol=1e-12)

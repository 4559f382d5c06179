"""Weighted graphs on the GPU (positive integer arc weights).

A level is a distance value: the forward sweep settles vertices one distance at
a time, which is the order of the reference's heap Dijkstra (relax.py:75-101,
oracle.py:44-61).  Golden vectors come from the reference package itself
(tests/golden/gen_golden_weighted.py): its weighted-tie fixture w5, weighted
members of its acceptance-corpus family and weighted grids -- Brandes dist /
sigma / delta per source, ``run_bc`` BC and the bsp-baseline per-source reports.
Larger seeded graphs are compared with the C oracle's Dijkstra.
"""

import json
import os
import random

import numpy as np
import pytest

import oracle as O
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_BSP, MODE_DIRECT

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-9, 1e-12
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def weighted_golden():
    with open(os.path.join(HERE, "golden", "reference_vectors_weighted.json")) as fh:
        return json.load(fh)


def graph_of(rec):
    return P.from_edges(rec["n"], [tuple(e) for e in rec["edges"]])


def with_weights(g, seed, wmax):
    """The same edges with seeded integer weights in [1, wmax] (equal on both arcs of an edge)."""
    rng = np.random.default_rng(seed)
    src, dst = g.arc_src, g.arc_dst
    keep = src < dst
    w = rng.integers(1, wmax + 1, size=int(keep.sum()))
    return P.from_edge_arrays(g.num_vertices, src[keep], dst[keep], w)


def test_w5_known_answer():
    # reference pkg/tests/test_oracle.py:31-34
    g = P.from_edges(5, [(0, 1, 2), (0, 2, 1), (1, 2, 1), (1, 3, 3), (2, 3, 4), (3, 4, 1)])
    with Engine(g) as e:
        dist, sigma, _ = e.debug_sources([0])
    assert dist[0].tolist() == [0, 2, 1, 5, 6]
    assert sigma[0].tolist() == [1, 2, 1, 3, 3]


def test_weighted_golden_vectors(weighted_golden):
    for rec in weighted_golden["graphs"]:
        g = graph_of(rec)
        srcs = [s["s"] for s in rec["sources"]]
        with Engine(g) as e:
            dist, sigma, delta = e.debug_sources(srcs)
            bc_all, st = e.run(list(range(rec["n"])))
            e.set_partition(2, rec["assignment"])
            bc_bsp, _ = e.run(rec["run_bc_sources"], MODE_BSP)
            reports = e.reports(len(rec["run_bc_sources"]))
        for i, sr in enumerate(rec["sources"]):
            assert dist[i].tolist() == sr["dist"], (rec["name"], sr["s"])
            assert sigma[i].tolist() == sr["sigma"], (rec["name"], sr["s"])
            assert np.allclose(delta[i], sr["delta"], rtol=RTOL, atol=ATOL), (rec["name"], sr["s"])
        assert np.allclose(bc_all, rec["bc_all_sources"], rtol=RTOL, atol=ATOL), rec["name"]
        assert np.allclose(bc_bsp, rec["run_bc_bsp_baseline"], rtol=RTOL, atol=ATOL), rec["name"]
        assert np.allclose(bc_bsp, rec["run_bc_hybir"], rtol=RTOL, atol=ATOL), rec["name"]   # modes agree in the reference
        for r, want in zip(reports, rec["per_source_bsp_baseline"]):
            it, ce, ml0, ml1, se, cb, l0, l1 = (int(x) for x in r)
            assert it == want["forward"]["supersteps"], rec["name"]
            assert ce == want["forward"]["comm_events"], rec["name"]
            assert [ml0, ml1] == want["forward"]["max_level"], rec["name"]
            assert se == want["backward"]["sync_events"], rec["name"]
            assert cb == want["backward"]["comm_bytes"], rec["name"]
            assert [l0, l1] == want["backward"]["levels"], rec["name"]


def test_run_bc_on_weighted_graphs(weighted_golden):
    rec = weighted_golden["graphs"][3]
    g = graph_of(rec)
    part = P.Partition(np.asarray(rec["assignment"], dtype=np.int32), 0.5, 2)
    res = P.run_bc(g, P.RunConfig(sources=rec["run_bc_sources"], mode="bsp-baseline", partition=part))
    assert np.allclose(res.bc, rec["run_bc_bsp_baseline"], rtol=RTOL, atol=ATOL)
    got = [p["forward"]["supersteps"] for p in res.per_source]
    assert got == [p["forward"]["supersteps"] for p in rec["per_source_bsp_baseline"]]
    res = P.run_bc(g, P.RunConfig(sources=rec["run_bc_sources"], mode="direct"))
    assert np.allclose(res.bc, rec["run_bc_bsp_baseline"], rtol=RTOL, atol=ATOL)
    res = P.run_bc(g, P.RunConfig(sources=rec["run_bc_sources"], mode="hybir", partition=part))
    assert np.allclose(res.bc, rec["run_bc_hybir"], rtol=RTOL, atol=ATOL)
    assert res.per_source == rec["per_source_hybir"]


def test_weighted_hybir_mode_matches_reference(weighted_golden):
    # the paper's border-matrix forward phase on weighted graphs (forward.py:188-256 with weighted
    # cut arcs and border tables): BC and every per-source report counter equal the reference's
    from paper_2008_05718_b200._capi import MODE_HYBIR
    for rec in weighted_golden["graphs"]:
        g = graph_of(rec)
        srcs = rec["run_bc_sources"]
        with Engine(g) as e:
            e.set_partition(2, rec["assignment"])
            assert e.border_counts(2).tolist() == [len(b) for b in rec["borders"]], rec["name"]
            bc, st = e.run(srcs, MODE_HYBIR)
            reports = e.reports(len(srcs))
            dist, sigma, delta = e.debug_sources(srcs[:32], MODE_HYBIR)
        assert np.allclose(bc, rec["run_bc_hybir"], rtol=RTOL, atol=ATOL), rec["name"]
        by_source = {sr["s"]: sr for sr in rec["sources"]}
        for i, s in enumerate(srcs[:32]):
            assert dist[i].tolist() == by_source[s]["dist"], (rec["name"], s)
            assert sigma[i].tolist() == by_source[s]["sigma"], (rec["name"], s)
            assert np.allclose(delta[i], by_source[s]["delta"], rtol=RTOL, atol=ATOL), (rec["name"], s)
        for r, want in zip(reports, rec["per_source_hybir"]):
            it, ce, ml0, ml1, se, cb, l0, l1 = (int(x) for x in r)
            assert it == want["forward"]["iterations"], rec["name"]
            assert ce == want["forward"]["comm_events"], rec["name"]
            assert [ml0, ml1] == want["forward"]["max_level"], rec["name"]
            assert se == want["backward"]["sync_events"], rec["name"]
            assert cb == want["backward"]["comm_bytes"], rec["name"]
            assert [l0, l1] == want["backward"]["levels"], rec["name"]


@pytest.mark.parametrize("case", ["rc", "rmat_hubs", "grid", "two_components"])
def test_weighted_seeded_graphs_vs_oracle(case):
    if case == "rc":
        g = with_weights(G.random_connected(600, 900, seed=11), 1, 10)
        srcs = list(range(0, 600, 7))
    elif case == "rmat_hubs":
        g = with_weights(G.rmat(12, 16, 5), 2, 4)          # hubs: sliced adjacency + hub kernel
        srcs = sorted(random.Random(3).sample(range(g.num_vertices), 70))
    elif case == "grid":
        g = with_weights(G.grid(30, 20), 3, 3)
        srcs = list(range(0, 600, 17))
    else:
        a = with_weights(G.random_connected(40, 30, seed=2), 4, 9)
        src, dst, w = a.arc_src, a.arc_dst, a.arc_weight
        keep = src < dst
        g = P.from_edge_arrays(90, np.concatenate([src[keep], src[keep] + 45]),
                               np.concatenate([dst[keep], dst[keep] + 45]), np.concatenate([w[keep], w[keep]]))
        srcs = [0, 5, 44, 45, 60, 88, 89]                   # vertices 40..44 and 85..89 are isolated
    assert not g.unit_weight
    with Engine(g) as e:
        e.set_option("groups", 2)
        e.set_option("item_arcs", 64)
        dist, sigma, delta = e.debug_sources(srcs[:40])
        bc, st = e.run(srcs)
    for i, s in enumerate(srcs[:40]):
        od, osg, odl, info = O.brandes_single_source(g, int(s))
        assert info["sigma_max"] < 2.0 ** 53
        assert np.array_equal(dist[i], od), (case, s)
        assert np.array_equal(sigma[i], osg), (case, s)
        assert np.allclose(delta[i], odl, rtol=RTOL, atol=ATOL), (case, s)
    obc, info = O.brandes_bc(g, srcs)
    assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL)
    assert st["max_levels"] == info["max_levels"]
    assert st["reached"] == info["reached"] and st["dag_arcs"] == info["dag_arcs"]


def test_all_ones_weights_take_the_unit_path():
    g = G.rmat(10, 8, 4)
    src, dst = g.arc_src, g.arc_dst
    keep = src < dst
    gw = P.from_edge_arrays(g.num_vertices, src[keep], dst[keep], np.ones(int(keep.sum()), dtype=np.int64))
    srcs = list(range(0, 1024, 9))
    with Engine(g) as e:
        a, _ = e.run(srcs)
    with Engine(gw) as e:
        b, _ = e.run(srcs)
    assert np.array_equal(a, b)


def test_reference_acceptance_corpus_on_the_gpu():
    """The reference's own acceptance gate (pkg/tests/test_acceptance.py: 200 seeded graphs, every
    second one weighted, 5 sources each) through the GPU engine in both partitioned modes: BC
    within 1e-9 of the reference's and every per-source report counter equal."""
    from paper_2008_05718_b200._capi import MODE_HYBIR
    with open(os.path.join(HERE, "golden", "acceptance_corpus.json")) as fh:
        doc = json.load(fh)
    assert len(doc["records"]) == 200
    for rec in doc["records"]:
        g = G.random_connected(rec["n"], rec["extra"], seed=1000 + rec["i"], weighted=rec["weighted"])
        assignment = np.array([int(c) for c in rec["assignment"]], dtype=np.int32)
        with Engine(g) as e:
            e.set_option("groups", 1)
            e.set_partition(2, assignment)
            bc_h, _ = e.run(rec["sources"], MODE_HYBIR)
            rep_h = e.reports(len(rec["sources"])).tolist()
            bc_b, _ = e.run(rec["sources"], MODE_BSP)
            rep_b = e.reports(len(rec["sources"])).tolist()
        assert np.allclose(bc_h, rec["bc"], rtol=RTOL, atol=ATOL), rec["i"]
        assert np.allclose(bc_b, rec["bc"], rtol=RTOL, atol=ATOL), rec["i"]
        assert rep_h == rec["hybir"], rec["i"]
        assert rep_b == rec["bsp"], rec["i"]


# ---- general positive integer weights: label-correcting distances + dependency-counted sweeps
# (csrc/bc_sssp.cuh).  The same oracle, the same bars: dist and sigma exact, delta / BC to 1e-9.

def check_against_oracle(g, srcs, e, n_inspect=40):
    dist, sigma, delta = e.debug_sources(srcs[:n_inspect])
    bc, st = e.run(srcs)
    for i, s in enumerate(srcs[:n_inspect]):
        od, osg, odl, info = O.brandes_single_source(g, int(s))
        assert info["sigma_max"] < 2.0 ** 53
        assert np.array_equal(dist[i], od), s
        assert np.array_equal(sigma[i], osg), s
        assert np.allclose(delta[i], odl, rtol=RTOL, atol=ATOL), s
    obc, info = O.brandes_bc(g, srcs)
    assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL)
    assert st["reached"] == info["reached"] and st["dag_arcs"] == info["dag_arcs"]
    return st


@pytest.mark.parametrize("case", ["rc", "rmat_hubs", "grid", "two_components"])
def test_general_weight_sweeps_on_small_weights(case):
    # the graphs of test_weighted_seeded_graphs_vs_oracle, forced onto the general-weight path
    if case == "rc":
        g = with_weights(G.random_connected(600, 900, seed=11), 1, 10)
        srcs = list(range(0, 600, 7))
    elif case == "rmat_hubs":
        g = with_weights(G.rmat(12, 16, 5), 2, 4)
        srcs = sorted(random.Random(3).sample(range(g.num_vertices), 70))
    elif case == "grid":
        g = with_weights(G.grid(30, 20), 3, 3)
        srcs = list(range(0, 600, 17))
    else:
        a = with_weights(G.random_connected(40, 30, seed=2), 4, 9)
        src, dst, w = a.arc_src, a.arc_dst, a.arc_weight
        keep = src < dst
        g = P.from_edge_arrays(90, np.concatenate([src[keep], src[keep] + 45]),
                               np.concatenate([dst[keep], dst[keep] + 45]), np.concatenate([w[keep], w[keep]]))
        srcs = [0, 5, 44, 45, 60, 88, 89]
    with Engine(g) as e:
        e.set_option("groups", 2)
        e.set_option("sssp", 1)
        check_against_oracle(g, srcs, e, n_inspect=len(srcs))   # partial last batches: pair-per-thread rounds
        e.set_option("sssp", 0)           # and the level-per-distance kernels give the same BC
        bc_levels, _ = e.run(srcs)
        e.set_option("sssp", 1)
        bc_general, _ = e.run(srcs)
    assert np.allclose(bc_levels, bc_general, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("case", ["road", "rc", "ties"])
def test_large_weights_vs_oracle(case):
    # DIMACS-style weights (no option set: the engine picks the general-weight sweeps)
    if case == "road":
        g = with_weights(G.road_like(40, 30, seed=3), 5, 200000)
        srcs = list(range(0, 1200, 23))
    elif case == "rc":
        g = with_weights(G.random_connected(500, 1500, seed=7), 6, 10 ** 6)
        srcs = list(range(0, 500, 5))
    else:
        # many equal-length paths under large weights: every edge weighs 5000
        base = G.grid(20, 15)
        src, dst = base.arc_src, base.arc_dst
        keep = src < dst
        g = P.from_edge_arrays(300, src[keep], dst[keep], np.full(int(keep.sum()), 5000, dtype=np.int64))
        srcs = list(range(0, 300, 7))
    assert int(g.arc_weight.max()) > 4096
    with Engine(g) as e:
        e.set_option("groups", 2)
        st = check_against_oracle(g, srcs, e)
    assert st["max_levels"] >= 2


def test_general_weight_sweeps_on_the_reference_golden_vectors(weighted_golden):
    for rec in weighted_golden["graphs"]:
        g = graph_of(rec)
        srcs = [s["s"] for s in rec["sources"]]
        with Engine(g) as e:
            e.set_option("sssp", 1)
            dist, sigma, delta = e.debug_sources(srcs)
            bc_all, _ = e.run(list(range(rec["n"])))
        for i, sr in enumerate(rec["sources"]):
            assert dist[i].tolist() == sr["dist"], (rec["name"], sr["s"])
            assert sigma[i].tolist() == sr["sigma"], (rec["name"], sr["s"])
            assert np.allclose(delta[i], sr["delta"], rtol=RTOL, atol=ATOL), (rec["name"], sr["s"])
        assert np.allclose(bc_all, rec["bc_all_sources"], rtol=RTOL, atol=ATOL), rec["name"]


def test_large_weights_through_run_bc_and_the_dimacs_loader(tmp_path):
    # a DIMACS .gr file with road-style weights (graph.py:139-173) through the public call; the
    # default partitioned mode steps down to 'direct' with a warning, a partitioned C call is refused
    g0 = with_weights(G.road_like(24, 24, seed=9), 8, 50000)
    src, dst, w = g0.arc_src, g0.arc_dst, g0.arc_weight
    path = tmp_path / "road.gr"
    with open(path, "w") as fh:
        fh.write("c test graph\np sp %d %d\n" % (g0.num_vertices, len(src)))
        for u, v, x in zip(src.tolist(), dst.tolist(), w.tolist()):
            fh.write("a %d %d %d\n" % (u + 1, v + 1, x))
    g = P.load_dimacs_gr(str(path))
    assert g.num_edges == g0.num_edges and int(g.arc_weight.max()) > 4096
    srcs = list(range(0, g.num_vertices, 11))
    obc, _ = O.brandes_bc(g, srcs)
    with pytest.warns(UserWarning, match="running mode 'direct'"):
        res = P.run_bc(g, P.RunConfig(sources=srcs))
    assert np.allclose(res.bc, obc, rtol=RTOL, atol=ATOL)
    res = P.run_bc(g, P.RunConfig(sources=srcs, mode="direct"))
    assert np.allclose(res.bc, obc, rtol=RTOL, atol=ATOL)
    with Engine(g) as e:
        e.set_partition(2, (np.arange(g.num_vertices) % 2).astype(np.int32))
        with pytest.raises(P.InputError, match="BC_MODE_DIRECT only"):
            e.run(srcs, MODE_BSP)


def test_general_weight_sweeps_deeper_than_one_flag_epoch():
    # a weighted path: the shortest-path DAG is ~20,000 arcs deep, beyond the 16,384 rounds one
    # epoch of round flags covers (engine_sssp.cuh: sssp_rounds restarts its round index)
    g = with_weights(G.path(20000), 12, 50000)
    srcs = [0, 7, 19999]
    with Engine(g) as e:
        st = check_against_oracle(g, srcs, e)
    assert st["max_levels"] > 16384

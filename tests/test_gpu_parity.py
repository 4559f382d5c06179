"""Parity of the CUDA path (through the C ABI) with the reference.

Bar (BASELINE.json north star): distances and path counts bit-exact, delta and
BC within 1e-9 relative in fp64.  Checked against (a) golden vectors produced
by the reference package, (b) the C oracle on seeded inputs, (c) properties
that hold at any size.
"""

import numpy as np
import pytest

import oracle as O
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_BSP, MODE_DIRECT, MODE_HYBIR

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-9, 1e-12   # the reference's own acceptance tolerance (test_acceptance.py:33,65-66)


def assert_sources_match_oracle(g, sources, dist, sigma, delta):
    for i, s in enumerate(sources):
        od, osg, odl, info = O.brandes_single_source(g, int(s))
        assert info["sigma_max"] < 2.0 ** 53
        assert np.array_equal(dist[i], od), "dist differs for source %d" % s
        assert np.array_equal(sigma[i], osg), "sigma differs for source %d" % s
        assert np.allclose(delta[i], odl, rtol=RTOL, atol=ATOL), "delta differs for source %d" % s


def test_golden_vectors_direct(golden_graphs):
    for name, (g, rec) in golden_graphs.items():
        srcs = [s["s"] for s in rec["sources"]]
        with Engine(g) as e:
            dist, sigma, delta = e.debug_sources(srcs)
            bc_all, _ = e.run(list(range(g.num_vertices)))
            bc_sub, _ = e.run(rec["run_bc_sources"])
        for i, s in enumerate(rec["sources"]):
            assert dist[i].tolist() == s["dist"], name
            assert sigma[i].tolist() == [float(x) for x in s["sigma"]], name
            assert np.allclose(delta[i], s["delta"], rtol=RTOL, atol=ATOL), name
        assert np.allclose(bc_all, rec["bc_all_sources"], rtol=RTOL, atol=ATOL), name
        assert np.allclose(bc_sub, rec["run_bc_hybir"], rtol=RTOL, atol=ATOL), name


def test_known_answers_through_run_bc():
    # reference pkg/tests/test_engine.py:14-17 and test_oracle.py:37-42
    cases = [
        (G.path(4), [0, 4, 4, 0]),
        (P.from_edges(4, [(0, 1, 1), (0, 2, 1), (1, 3, 1), (2, 3, 1)]), [1, 1, 1, 1]),
        (P.from_edges(6, [(i, (i + 1) % 6, 1) for i in range(6)]), [4] * 6),
        (P.from_edges(4, [(i, j, 1) for i in range(4) for j in range(i + 1, 4)]), [0] * 4),
        (P.from_edges(5, [(0, i, 1) for i in range(1, 5)]), [12, 0, 0, 0, 0]),
    ]
    for g, want in cases:
        res = P.run_bc(g, P.RunConfig(mode="direct"))
        assert np.allclose(res.bc, want, rtol=RTOL, atol=ATOL)
        assert res.mteps > 0 and res.elapsed > 0


@pytest.mark.parametrize("seed", range(6))
def test_random_graphs_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 400))
    g = G.random_connected(n, int(rng.integers(0, 2 * n)), seed=seed)
    srcs = rng.choice(n, size=min(n, 70), replace=False).tolist()
    with Engine(g) as e:
        e.set_option("groups", int(rng.integers(1, 4)))
        dist, sigma, delta = e.debug_sources(srcs)
        bc, st = e.run(srcs)
    assert_sources_match_oracle(g, srcs, dist, sigma, delta)
    obc, info = O.brandes_bc(g, srcs)
    assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL)
    assert (st["reached"], st["arcs_reached"], st["dag_arcs"]) == (
        info["reached"], info["arcs_reached"], info["dag_arcs"])
    assert st["max_levels"] == info["max_levels"]


def test_config1_rmat12_all_sources(rmat12):
    """BASELINE config 1: R-MAT scale-12 EF-8, all 4096 sources."""
    g = rmat12
    srcs = list(range(g.num_vertices))
    with Engine(g) as e:
        e.set_option("groups", 16)
        bc, st = e.run(srcs)
        sample = list(range(0, g.num_vertices, 41))
        dist, sigma, delta = e.debug_sources(sample)
    obc, info = O.brandes_bc(g, srcs)
    assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL)
    assert st["reached"] == info["reached"] and st["dag_arcs"] == info["dag_arcs"]
    assert_sources_match_oracle(g, sample, dist, sigma, delta)
    # bc max=1.482890e+06 sum=1.623059e+07 on this graph
    assert bc.max() == pytest.approx(1.482890e6, rel=1e-6)
    assert bc.sum() == pytest.approx(1.623059e7, rel=1e-6)


def test_hub_slices_and_item_sizes():
    # hubs (degree >> item_arcs) take the sliced path; results must not depend
    # on how the adjacency is cut into work items
    g = G.rmat(13, 16, 3)
    srcs = list(range(0, g.num_vertices, 97))
    ref = None
    for item_arcs in (32, 64, 256, 1024):
        with Engine(g) as e:
            e.set_option("item_arcs", item_arcs)
            dist, sigma, delta = e.debug_sources(srcs[:40])
            bc, _ = e.run(srcs)
        assert_sources_match_oracle(g, srcs[:40], dist, sigma, delta)
        if ref is None:
            ref = bc
            obc, _ = O.brandes_bc(g, srcs)
            assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL)
        else:
            assert np.allclose(bc, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("b", [1, 7, 8, 9, 31, 32, 33, 40, 64, 65, 100])
def test_staged_gather_round_boundaries(b):
    # complete bipartite K_{a,b}: from a source in A every other vertex of A has all b vertices
    # of B as parents, so the 32-arc slices of the level kernel carry b mod 32 (or 32) hit arcs --
    # every fill of the staged hit-arc list around the round sizes (4 backward, 8 forward) and
    # its padding; sources in B give single-hit slices.  sparse = 0 keeps every level on the
    # dense pull kernel.
    a = 6
    edges = [(i, a + j, 1) for i in range(a) for j in range(b)]
    g = P.from_edges(a + b, edges)
    srcs = list(range(a + b))
    for sparse, row_cache in ((0, 1), (0, 0), (1, -1)):   # row_cache 0: gathers bypass L1
        with Engine(g) as e:
            e.set_option("sparse", sparse)
            e.set_option("row_cache", row_cache)
            dist, sigma, delta = e.debug_sources(srcs)
            bc, _ = e.run(srcs)
        assert_sources_match_oracle(g, srcs, dist, sigma, delta)
        assert np.allclose(bc, O.brandes_bc(g, srcs)[0], rtol=RTOL, atol=ATOL)


def test_edge_cases():
    # single vertex, isolated sources, duplicate sources, empty source list,
    # disconnected components, partial last group
    one = P.from_edges(1, [])
    with Engine(one) as e:
        bc, st = e.run([0])
        assert bc.tolist() == [0.0] and st["reached"] == 1
        d, s, dl = e.debug_sources([0])
        assert d.tolist() == [[0]] and s.tolist() == [[1.0]] and dl.tolist() == [[0.0]]
    g = P.from_edges(7, [(0, 1, 1), (1, 2, 1), (4, 5, 1)])      # 3 and 6 isolated
    with Engine(g) as e:
        bc, _ = e.run([])
        assert not bc.any()
        bc, _ = e.run([3, 6])
        assert not bc.any()
        bc1, _ = e.run([0, 2, 4])
        bc2, _ = e.run([0, 2, 4, 0, 2, 4])
        assert np.allclose(2 * bc1, bc2)
        d, s, dl = e.debug_sources([0, 3])
        assert d[0].tolist() == [0, 1, 2, -1, -1, -1, -1] and d[1].tolist() == [-1, -1, -1, 0, -1, -1, -1]
        assert s[1].tolist() == [0, 0, 0, 1, 0, 0, 0]
        with pytest.raises(P.InputError):
            e.run([7])
        with pytest.raises(P.InputError):
            e.run([-1])
        with pytest.raises(P.InputError):
            e.set_option("groups", 0)
    srcs = list(range(45))                                       # 32 + 13 lanes
    g = G.grid(9, 5)
    with Engine(g) as e:
        e.set_option("groups", 1)
        bc, _ = e.run(srcs)
    assert np.allclose(bc, O.brandes_bc(g, srcs)[0], rtol=RTOL, atol=ATOL)


def test_deep_graph_path_and_grid():
    # high diameter: many levels, speculative level launches, sigma stays small
    p = G.path(3000)
    with Engine(p) as e:
        bc, st = e.run([0, 1500, 2999])
    assert st["max_levels"] == 3000
    assert np.allclose(bc, O.brandes_bc(p, [0, 1500, 2999])[0], rtol=RTOL, atol=ATOL)
    r = G.road_like(96, 96, keep=0.2, seed=1)
    srcs = list(range(0, r.num_vertices, 211))
    with Engine(r) as e:
        dist, sigma, delta = e.debug_sources(srcs[:8])
        bc, _ = e.run(srcs)
    for i, s in enumerate(srcs[:8]):
        od, osg, odl, info = O.brandes_single_source(r, s)
        assert np.array_equal(dist[i], od)
        if info["sigma_max"] < 2.0 ** 53:
            assert np.array_equal(sigma[i], osg)
        else:   # beyond exact integers: fp64 path counts, 1e-12 relative (SURVEY.md hard part 1)
            assert np.allclose(sigma[i], osg, rtol=1e-12)
        assert np.allclose(delta[i], odl, rtol=RTOL, atol=ATOL)
    assert np.allclose(bc, O.brandes_bc(r, srcs)[0], rtol=RTOL, atol=ATOL)


def test_persistent_sweeps_equal_level_by_level():
    # runs of thin levels inside one cooperative launch (bc_deep.cuh) against one launch per level
    cases = [(G.path(2500), [0, 17, 1250, 2499]),                 # > 1024 levels: several launches
             (G.road_like(80, 80, keep=0.2, seed=5), list(range(0, 6400, 61))),
             (G.grid(40, 25), list(range(0, 1000, 7)))]
    for g, srcs in cases:
        out = {}
        for deep in (0, 1):
            with Engine(g) as e:
                e.set_option("deep", deep)
                e.set_option("groups", 2)
                d, s, dl = e.debug_sources(srcs[:20])
                bc, st = e.run(srcs)
            out[deep] = (d, s, dl, bc, st)
        assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
        assert np.array_equal(out[0][2], out[1][2])          # same arithmetic, same order
        assert np.allclose(out[0][3], out[1][3], rtol=1e-12, atol=1e-12)
        for key in ("reached", "arcs_reached", "dag_arcs", "max_levels"):
            assert out[0][4][key] == out[1][4][key], key
        assert out[1][4]["launches"] < out[0][4]["launches"]
        assert np.allclose(out[1][3], O.brandes_bc(g, srcs)[0], rtol=RTOL, atol=ATOL)


def test_device_block_cache_reuse_and_release(rmat12):
    # closed engines leave their device blocks in the per-device cache: the next engine takes
    # them over (dirty), a release hands them back to the driver; results never change
    from paper_2008_05718_b200 import _capi
    srcs = list(range(0, 4096, 5))
    small = G.grid(9, 5)
    with Engine(rmat12) as e:
        e.set_option("bwd_push", 0)          # bit-for-bit comparisons below: sums in arc order
        first, _ = e.run(srcs)
    for _ in range(2):
        with Engine(small) as e:
            bc_small, _ = e.run(list(range(45)))
        with Engine(rmat12) as e:
            e.set_option("bwd_push", 0)
            again, _ = e.run(srcs)
        assert np.array_equal(first, again)
        assert np.allclose(bc_small, O.brandes_bc(small, list(range(45)))[0], rtol=RTOL, atol=ATOL)
        _capi.release_cached_memory()
    with Engine(rmat12) as e:
        e.set_option("bwd_push", 0)
        assert np.array_equal(first, e.run(srcs)[0])


def test_deterministic_and_linear(rmat12):
    g = rmat12
    a = list(range(0, 4096, 9))
    b = list(range(1, 4096, 13))
    with Engine(g) as e:
        e.set_option("bwd_push", 0)      # every backward level parent-driven: sums in CSR arc order
        bc_a, _ = e.run(a)
        bc_a2, _ = e.run(a)
        bc_b, _ = e.run(b)
        bc_ab, _ = e.run(a + b)
    assert np.array_equal(bc_a, bc_a2)                       # bit-reproducible
    with Engine(g) as e:                 # default: child-driven levels add in atomic order
        bc_d, _ = e.run(a)
    assert np.allclose(bc_d, bc_a, rtol=1e-12, atol=1e-9)
    assert np.allclose(bc_a + bc_b, bc_ab, rtol=1e-12)       # BC is a sum over sources
    assert bc_ab.min() >= 0.0


@pytest.mark.slow
def test_config2_rmat20_sample():
    """BASELINE config 2 at full size: R-MAT scale-20 EF-16; oracle on a 48-source sample,
    size-independent properties on the full 1024-source run."""
    import random
    g = G.rmat(20, 16, 1)
    assert g.num_vertices == 1 << 20
    srcs = sorted(random.Random(0).sample(range(g.num_vertices), 1024))
    with Engine(g) as e:
        e.set_option("groups", 8)
        bc, st = e.run(srcs)
        bc48, _ = e.run(srcs[:48])
        dist, sigma, delta = e.debug_sources(srcs[:4])
    obc, info = O.brandes_bc(g, srcs[:48])
    assert np.allclose(bc48, obc, rtol=RTOL, atol=ATOL)
    assert_sources_match_oracle(g, srcs[:4], dist, sigma, delta)
    # sum over v of delta_s[v] = sum over reached t != s of (dist(s,t) - 1) for every source,
    # so the BC total is fixed by the distance histogram alone
    total = 0
    for i in range(4):
        d = dist[i][dist[i] > 0]
        assert delta[i].sum() - delta[i][srcs[i]] == pytest.approx(float((d - 1).sum()), rel=1e-9)
    deg = np.diff(g.offsets)
    assert not bc[deg == 0].any() and bc.min() >= 0.0
    assert st["sources"] == 1024 and st["max_levels"] >= 5


def test_level_ordered_backward_of_deep_graphs():
    """Deep graphs sweep backward over level-ordered sigma / coef values (deep_backward_compact_kernel):
    same BC as the row layout, with per-group BC partials (deep_compact = 2) and with the atomically
    updated BC vector (deep_compact = 1, the default)."""
    cases = [(G.path(2500), [0, 17, 1250, 2499] + list(range(3, 2500, 97))),
             (G.road_like(96, 96, keep=0.2, seed=5), list(range(0, 9216, 41))),
             (G.grid(48, 30), list(range(0, 1440, 7)))]
    for g, srcs in cases:
        out = {}
        for mode in (0, 1, 2):
            with Engine(g) as e:
                e.set_option("groups", 3)
                e.set_option("deep_compact", mode)
                bc, st = e.run(srcs)
                bc2, _ = e.run(srcs)           # a second run on the same handle (buffers reused)
            out[mode] = (bc, st)
            assert np.allclose(bc, bc2, rtol=1e-12, atol=1e-12)
        # (path counts are added with atomics on every path: exact below 2^53, rounding order above)
        assert np.allclose(out[0][0], out[2][0], rtol=1e-12, atol=1e-9)
        assert np.allclose(out[0][0], out[1][0], rtol=1e-12, atol=1e-9)
        obc, _ = O.brandes_bc(g, srcs)
        assert np.allclose(out[1][0], obc, rtol=RTOL, atol=ATOL)
    # the partitioned sweeps on frontier queues take the same path
    g = G.road_like(64, 64, keep=0.2, seed=3)
    srcs = list(range(0, 4096, 29))
    part = P.strip_partition(64, 64, 4)
    res = {}
    for mode in (0, 1):
        with Engine(g) as e:
            e.set_option("groups", 2)
            e.set_option("reports", 0)
            e.set_option("deep_compact", mode)
            e.set_partition(4, part.assignment)
            res[mode], _ = e.run(srcs, MODE_HYBIR)
    assert np.allclose(res[0], res[1], rtol=1e-12, atol=1e-9)
    assert np.allclose(res[1], O.brandes_bc(g, srcs)[0], rtol=RTOL, atol=ATOL)


def test_level_ordered_sweeps_edge_cases():
    """Level-ordered deep sweeps with awkward source lists: duplicates (two lanes of one group on
    the same vertex), isolated sources, sources in different components, a single source, none."""
    from paper_2008_05718_b200 import from_edge_arrays
    base = G.road_like(64, 64, keep=0.2, seed=7)
    # two disjoint copies + a few isolated vertices
    n0 = base.num_vertices
    und = base.arc_src < base.arc_dst
    u = np.concatenate([base.arc_src[und], base.arc_src[und] + n0])
    v = np.concatenate([base.arc_dst[und], base.arc_dst[und] + n0])
    g = from_edge_arrays(2 * n0 + 5, u, v)
    iso = 2 * n0 + 2
    for srcs in ([5, 5, 900, n0 + 17, iso, 5, 4000, n0 + 4000, iso, 77],
                 [123], [iso], [], list(range(0, 2 * n0, 257)) + [iso]):
        obc, _ = O.brandes_bc(g, srcs)
        for mode in (1, 0):
            with Engine(g) as e:
                e.set_option("groups", 2)
                e.set_option("deep_compact", mode)
                bc, st = e.run(srcs)
            assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL), (srcs[:4], mode)
            assert st["sources"] == len(srcs)
    # the same through the partitioned mode (isolated and duplicate sources keep their lanes there)
    part = P.Partition((np.arange(g.num_vertices) >= n0).astype(np.int32), 0.5, 2)   # no cut edges at all
    strips = P.Partition(((np.arange(g.num_vertices) % n0) // (n0 // 2) % 2).astype(np.int32), 0.5, 2)
    srcs = [5, 5, 900, n0 + 17, iso, 4000, n0 + 4000, 77]
    obc, _ = O.brandes_bc(g, srcs)
    for p in (part, strips):
        with Engine(g) as e:
            e.set_option("groups", 1)
            e.set_option("reports", 0)
            e.set_partition(2, p.assignment)
            bc, _ = e.run(srcs, MODE_HYBIR)
        assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL)


def test_path_counts_beyond_2_53_against_the_bigint_reference():
    """sigma above 2^53 (SURVEY.md hard part 1) pinned to the reference's exact-integer oracle
    (golden vectors of tests/golden/gen_golden_bigsigma.py, 40 x 32 lattice, max sigma 2^66):
    distances exact, GPU path counts within 1e-12 relative, delta / BC within 1e-9."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bigsigma_vectors.npz"))
    g = G.grid(int(z["rows"]), int(z["cols"]))
    srcs = z["sources"].tolist()
    assert z["sigma_max_log2"].max() > 53
    with Engine(g) as e:
        dist, sigma, delta = e.debug_sources(srcs)
        bc, _ = e.run(srcs)
        e.set_option("sparse", 0)                      # dense pull levels only
        dist2, sigma2, delta2 = e.debug_sources(srcs)
    for d_, s_, dl_ in ((dist, sigma, delta), (dist2, sigma2, delta2)):
        assert np.array_equal(d_, z["dist"])
        assert np.allclose(s_, z["sigma"], rtol=1e-12, atol=0)
        assert np.allclose(dl_, z["delta"], rtol=RTOL, atol=ATOL)
    assert np.allclose(bc, z["bc"], rtol=RTOL, atol=ATOL)
    # the partitioned modes on the same graph (border tables hold path counts above 2^53 too)
    part = P.strip_partition(int(z["rows"]), int(z["cols"]), 2)
    for mode in (MODE_HYBIR, MODE_BSP):
        with Engine(g) as e:
            e.set_partition(2, part.assignment)
            e.set_option("reports", 0)
            bcp, _ = e.run(srcs, mode)
        assert np.allclose(bcp, z["bc"], rtol=RTOL, atol=ATOL), mode


@pytest.mark.slow
def test_config3_road2048_sample():
    """BASELINE config 3's graph at full size (road-like 2048 x 2048, ~4,100 levels, path counts far
    above 2^53) at a reduced source count: oracle port on a 4-source sample, direct == hybir in 8
    strips, and the distance-histogram identity on the inspected sources."""
    g = G.road_like(2048, 2048, keep=0.2, seed=1)
    assert g.num_vertices == 1 << 22
    srcs = pick = sorted(__import__("random").Random(0).sample(range(g.num_vertices), 64))
    with Engine(g) as e:
        e.set_option("groups", 2)
        bc, st = e.run(srcs)
        bc4, _ = e.run(pick[:4])
        dist, sigma, delta = e.debug_sources(pick[:2])
    obc, info = O.brandes_bc(g, pick[:4])
    assert info["sigma_max"] > 2.0 ** 53
    assert np.allclose(bc4, obc, rtol=RTOL, atol=ATOL)
    for i in range(2):
        od, osg, odl, _ = O.brandes_single_source(g, pick[i])
        assert np.array_equal(dist[i], od)
        assert np.allclose(sigma[i], osg, rtol=1e-12, atol=0)
        assert np.allclose(delta[i], odl, rtol=RTOL, atol=ATOL)
        d = dist[i][dist[i] > 0]
        assert delta[i].sum() - delta[i][pick[i]] == pytest.approx(float((d - 1).sum()), rel=1e-9)
    assert st["max_levels"] > 3000
    part = P.strip_partition(2048, 2048, 8)
    with Engine(g) as e:
        e.set_option("groups", 2)
        e.set_option("reports", 0)
        e.set_partition(8, part.assignment)
        bch, sth = e.run(srcs, MODE_HYBIR)
    assert np.allclose(bch, bc, rtol=RTOL, atol=ATOL)
    assert sth["iterations"] >= len(srcs)


@pytest.mark.slow
def test_config4_erdos_renyi_sample():
    """BASELINE config 4's graph at full size (Erdos-Renyi n = 2^22, average degree 32) at a reduced
    source count: oracle on a sample, linearity over a split of the source list."""
    g = G.erdos_renyi(1 << 22, 1 << 26, 1)
    srcs = sorted(__import__("random").Random(0).sample(range(g.num_vertices), 128))
    with Engine(g) as e:
        e.set_option("groups", 4)
        bc, st = e.run(srcs)
        bc_a, _ = e.run(srcs[:64])
        bc_b, _ = e.run(srcs[64:])
        bc8, _ = e.run(srcs[:8])
        dist, sigma, delta = e.debug_sources(srcs[:2])
    assert np.allclose(bc_a + bc_b, bc, rtol=1e-12, atol=1e-9)
    obc, info = O.brandes_bc(g, srcs[:8])
    assert info["sigma_max"] < 2.0 ** 53
    assert np.allclose(bc8, obc, rtol=RTOL, atol=ATOL)
    assert_sources_match_oracle(g, srcs[:2], dist, sigma, delta)
    assert 5 <= st["max_levels"] <= 12


def test_push_pull_switch_equivalence():
    # queue levels + top-down push (default) against dense pull only: same dist / sigma / BC
    cases = [G.rmat(13, 16, 3), G.road_like(64, 64, keep=0.2, seed=2), G.erdos_renyi(4000, 12000, 3)]
    for g in cases:
        rng = np.random.default_rng(9)
        srcs = rng.choice(g.num_vertices, size=70, replace=False).tolist()
        out = {}
        for sparse in (0, 1):
            with Engine(g) as e:
                e.set_option("sparse", sparse)
                e.set_option("groups", 2)
                d, s, dl = e.debug_sources(srcs[:33])
                bc, st = e.run(srcs)
            out[sparse] = (d, s, dl, bc, st)
        assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
        assert np.allclose(out[0][2], out[1][2], rtol=1e-12, atol=1e-12)
        assert np.allclose(out[0][3], out[1][3], rtol=1e-12, atol=1e-12)
        for key in ("reached", "arcs_reached", "dag_arcs", "max_levels"):
            assert out[0][4][key] == out[1][4][key], key
        assert_sources_match_oracle(g, srcs[:33], out[1][0], out[1][1], out[1][2])
        with Engine(g) as e:      # push at (almost) every level
            e.set_option("push_beta", 1)
            bc1, _ = e.run(srcs)
        assert np.allclose(bc1, out[0][3], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("case", ["rmat12", "rmat14_batches", "star_and_isolated", "small_forced"])
def test_degree_renumbered_sweeps(case):
    """Unpartitioned unit-weight runs of skewed graphs sweep a copy of the graph renumbered by
    descending degree (csrc/bc_relabel.cuh): sources are renamed on the way in, BC on the way
    out.  Same BC as on the caller's ids (and as the oracle), same traversal counters."""
    if case == "rmat12":
        g = G.rmat(12, 8, 1)
        srcs = list(range(0, 4096, 3))
        groups = 8
    elif case == "rmat14_batches":
        g = G.rmat(14, 16, 3)
        srcs = sorted(np.random.default_rng(4).choice(g.num_vertices, 300, replace=False).tolist())
        groups = 2                                  # several batches, the last one partial
    elif case == "star_and_isolated":
        # one hub, leaves, a tail, isolated vertices (also as sources)
        edges = [(0, i) for i in range(1, 200)] + [(200 + i, 201 + i) for i in range(20)] + [(5, 200)]
        g = P.from_edges(260, edges)
        srcs = [0, 1, 5, 199, 200, 220, 221, 259]
        groups = 1
    else:
        g = G.random_connected(300, 500, seed=5)
        srcs = list(range(0, 300, 2))
        groups = 2
    with Engine(g) as e:
        e.set_option("groups", groups)
        e.set_option("bwd_push", 0)                 # bc_ren == bc_ren2 bit for bit needs arc-order sums
        e.set_option("relabel", 0)
        bc_plain, st_plain = e.run(srcs)
        e.set_option("relabel", 1)
        bc_ren, st_ren = e.run(srcs)
        bc_ren2, _ = e.run(srcs)
        dist, sigma, delta = e.debug_sources(srcs[:8])      # inspection stays on the caller's ids
    obc, info = O.brandes_bc(g, srcs)
    assert np.allclose(bc_ren, obc, rtol=1e-9, atol=1e-12)
    assert np.allclose(bc_ren, bc_plain, rtol=1e-12, atol=1e-12)
    assert np.array_equal(bc_ren, bc_ren2)
    for key in ("reached", "arcs_reached", "dag_arcs", "max_levels"):
        assert st_ren[key] == st_plain[key], key
    assert st_ren["reached"] == info["reached"] and st_ren["dag_arcs"] == info["dag_arcs"]
    for i, s in enumerate(srcs[:8]):
        od, osg, odl, _ = O.brandes_single_source(g, int(s))
        assert np.array_equal(dist[i], od) and np.array_equal(sigma[i], osg)


def test_degree_renumbering_is_chosen_by_skew_and_work():
    # R-MAT (hubs) is renumbered by default once the handle has seen 2048 sources, a grid never:
    # the default run equals the forced one bit for bit when it applies and the plain one otherwise
    g = G.rmat(13, 16, 2)
    srcs = np.nonzero(np.diff(g.offsets) > 0)[0][:2100].tolist()     # (sources without arcs take no lane: not counted)
    with Engine(g) as e:
        e.set_option("bwd_push", 0)             # bit-for-bit comparisons
        first, _ = e.run(srcs[:200])            # 200 sources: not yet
        many, _ = e.run(srcs)                   # 2300 seen: renumbered from here on
        again, _ = e.run(srcs[:200])
        e.set_option("relabel", 0)
        plain_few, _ = e.run(srcs[:200])
        e.set_option("relabel", 1)
        forced_few, _ = e.run(srcs[:200])
        forced_many, _ = e.run(srcs)
    assert np.array_equal(first, plain_few)
    assert np.array_equal(again, forced_few)
    assert np.array_equal(many, forced_many)
    g = G.grid(40, 40)
    srcs = list(range(g.num_vertices))
    with Engine(g) as e:
        e.set_option("bwd_push", 0)
        e.run(srcs)
        default, _ = e.run(srcs)
        e.set_option("relabel", 0)
        plain, _ = e.run(srcs)
    assert np.array_equal(default, plain)


@pytest.mark.parametrize("case", ["rmat13", "rmat12_batches", "tree", "grid"])
def test_child_driven_backward_levels(case):
    """Direction switch of the dependency sweep (csrc/bc_bwd_push.cuh): past the peak level the
    children add their coef into their parents (atomic adds) instead of every parent scanning all
    its arcs (backward.py:95-103).  Same BC as the parent-driven sweep to rounding, same as the
    oracle within the 1e-9 of the specification; delta per source through the inspection path."""
    if case == "rmat13":
        g = G.rmat(13, 16, 5)
        srcs = np.nonzero(np.diff(g.offsets) > 0)[0][::7][:512].tolist()
        groups = 0
    elif case == "rmat12_batches":
        g = G.rmat(12, 8, 1)
        srcs = list(range(0, 4096, 3))
        groups = 4                              # several batches, the last one partial
    elif case == "tree":
        # a broom: long handle, then a wide fan -- levels shrink and grow by large factors
        edges = [(i, i + 1) for i in range(40)] + [(40, 41 + i) for i in range(600)]
        edges += [(41 + i, 641 + (i % 7)) for i in range(600)]
        g = P.from_edges(660, edges)
        srcs = list(range(0, 660, 5))
        groups = 0
    else:
        g = G.grid(24, 31)
        srcs = list(range(0, g.num_vertices, 3))
        groups = 0
    out = {}
    for beta in (0, 1, 4, 16):
        with Engine(g) as e:
            if groups:
                e.set_option("groups", groups)
            e.set_option("bwd_push", beta)
            out[beta] = e.run(srcs)
    obc, info = O.brandes_bc(g, srcs)
    for beta in (0, 1, 4, 16):
        bc, st = out[beta]
        assert np.allclose(bc, obc, rtol=RTOL, atol=ATOL), beta
        assert np.allclose(bc, out[0][0], rtol=1e-12, atol=1e-9), beta
        for key in ("reached", "arcs_reached", "dag_arcs", "max_levels"):
            assert st[key] == out[0][1][key], (beta, key)
    if case.startswith("rmat"):
        # the switch did fire on the small-world graphs: three launches per child-driven level
        assert out[1][1]["launches"] != out[0][1]["launches"]

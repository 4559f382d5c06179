"""Host-side logic: graph normalisation, partitioning, borders, source
selection and configuration errors -- the reference's behaviour for each is
cited next to the check."""

import os
import random

import numpy as np
import pytest

import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200.engine import default_groups, make_partition


def test_csr_of_p4():
    # reference pkg/tests/test_graph.py:12-18
    g = G.path(4)
    assert g.offsets.tolist() == [0, 1, 3, 5, 6]
    assert g.arc_src.tolist() == [0, 1, 1, 2, 2, 3]
    assert g.arc_dst.tolist() == [1, 0, 2, 1, 3, 2]
    assert g.num_edges == 3 and g.num_arcs == 6 and g.inf_distance == 4
    assert g.rev_arc.tolist() == [1, 0, 3, 2, 5, 4]


def test_from_edges_normalisation():
    # self loops dropped, parallel edges collapse to the minimum weight,
    # symmetrised (graph.py:64-110)
    g = P.from_edges(4, [(0, 1, 5), (1, 0, 2), (2, 2, 1), (3, 1, 7), (1, 3, 9)])
    assert g.num_edges == 2
    assert g.arc_src.tolist() == [0, 1, 1, 3] and g.arc_dst.tolist() == [1, 0, 3, 1]
    assert g.arc_weight.tolist() == [2, 2, 7, 7]
    assert g.inf_distance == 10 and not g.unit_weight
    assert P.from_edges(3, []).num_edges == 0


def test_from_edges_errors():
    with pytest.raises(P.FormatError):
        P.from_edges(3, [(0, 3, 1)])
    with pytest.raises(P.DomainError):
        P.from_edges(3, [(0, 1, -1)])
    with pytest.raises(P.DomainError):
        P.from_edges(3, [(0, 1, 0)])
    # the first offending edge decides, as in the reference's edge-by-edge loop
    with pytest.raises(P.DomainError):
        P.from_edges(3, [(0, 1, 0), (0, 9, 1)])
    assert issubclass(P.FormatError, P.InputError) and issubclass(P.InputError, P.HybirError)


def test_golden_graphs_round_trip(golden_graphs):
    for g, rec in golden_graphs.values():
        assert g.offsets.tolist() == rec["offsets"]
        assert g.arc_dst.tolist() == rec["arc_dst"]
        assert g.inf_distance == rec["inf"]


def test_borders_match_reference(golden_graphs):
    for g, rec in golden_graphs.values():
        p = P.Partition(np.asarray(rec["assignment"], dtype=np.int8), 0.5, 2)
        bs = P.identify_borders(g, p)
        assert [list(b) for b in bs.borders] == rec["borders"]
        assert [[u, v] for u, v, _ in bs.cut_arcs] == rec["cut_arcs"]
        for side in (0, 1):
            assert bs.index[side] == {v: i for i, v in enumerate(rec["borders"][side])}


def test_known_borders():
    # reference pkg/tests/test_partition.py:99-111
    g = G.path(4)
    bs = P.identify_borders(g, P.Partition(np.array([0, 0, 1, 1], dtype=np.int8)))
    assert bs.borders == ([1], [2]) and bs.cut_arcs == [(1, 2, 1), (2, 1, 1)]
    d = P.from_edges(4, [(0, 1, 1), (0, 2, 1), (1, 3, 1), (2, 3, 1)])
    bs = P.identify_borders(d, P.Partition(np.array([0, 0, 1, 1], dtype=np.int8)))
    assert bs.borders == ([0, 1], [2, 3]) and len(bs.cut_arcs) == 4


def test_greedy_bipartition_matches_reference(golden_graphs):
    # fixtures whose partition came from the reference's greedy_bipartition
    cases = {"grid9x7_greedy": (0.5, 3), "rc_n12_s1000": (0.7, 1000), "rc_n25_s1002": (0.5, 1002),
             "rc_n40_s1004": (0.5, 1004), "rc_n60_s1006": (0.7, 1006), "rc_n90_s1008": (0.5, 1008),
             "rmat8": (0.5, 0)}
    for name, (ratio, seed) in cases.items():
        g, rec = golden_graphs[name]
        p = P.greedy_bipartition(g, ratio, seed=seed)
        assert p.assignment.tolist() == rec["assignment"], name


def test_greedy_bipartition_errors():
    with pytest.raises(P.InputError):
        P.greedy_bipartition(G.path(4), 1.0)
    with pytest.raises(P.InputError):
        P.greedy_bipartition(P.from_edges(1, []), 0.5)


def test_rmat12_is_the_baseline_graph(rmat12):
    # n=4,096, m=26,603, 1,129 isolated, max degree 931,
    # greedy borders (780, 908), 4,060 cut arcs
    deg = np.diff(rmat12.offsets)
    assert (rmat12.num_vertices, rmat12.num_edges) == (4096, 26603)
    assert int((deg == 0).sum()) == 1129 and int(deg.max()) == 931
    p = P.greedy_bipartition(rmat12, 0.5, seed=0)
    bs = P.identify_borders(rmat12, p)
    assert bs.counts() == (780, 908) and len(bs.cut_src) == 4060


def test_kway_partitions():
    g = G.grid(8, 6)
    p = P.strip_partition(8, 6, 4)
    assert p.sizes == (12, 12, 12, 12)
    bs = P.identify_borders(g, p)
    assert bs.counts() == (6, 12, 12, 6)
    assert P.block_partition(g, 3).sizes == (16, 16, 16)
    assert P.single_partition(g).num_parts == 1
    assert P.identify_borders(g, P.single_partition(g)).counts() == (0,)


def test_select_sources_rule():
    g = G.path(50)
    assert P.select_sources(g, P.RunConfig()) == list(range(50))
    assert P.select_sources(g, P.RunConfig(sources=[7, 3, 3])) == [7, 3, 3]
    want = sorted(random.Random(5).sample(range(50), 10))     # engine.py:82-84
    assert P.select_sources(g, P.RunConfig(num_sources=10, seed=5)) == want
    assert len(P.select_sources(g, P.RunConfig(num_sources=99))) == 50
    with pytest.raises(P.InputError):
        P.select_sources(g, P.RunConfig(sources=[50]))


def test_run_config_validation():
    with pytest.raises(P.InputError):
        P.RunConfig(mode="nope")
    with pytest.raises(P.InputError):
        P.RunConfig(num_sources=0)
    with pytest.raises(P.InputError):
        P.RunConfig(backward_strategies=("vertex-pull", "sideways"))
    with pytest.raises(P.InputError):
        P.RunConfig(gpu_mode="ring")
    with pytest.raises(P.InputError):
        P.run_bc(P.from_edges(0, []), P.RunConfig())
    with pytest.raises(P.InputError):      # the multi-GPU border exchange is unit-weight
        P.run_bc(P.from_edges(3, [(0, 1, 2), (1, 2, 1)]),
                 P.RunConfig(num_gpus=2, gpu_mode="graph-partitioned"))


def test_make_partition_modes():
    g = G.grid(6, 6)
    assert make_partition(g, P.RunConfig(num_partitions=1)).num_parts == 1
    assert make_partition(g, P.RunConfig(mode="direct")).num_parts == 1
    assert make_partition(g, P.RunConfig()).num_parts == 2
    assert make_partition(g, P.RunConfig(num_partitions=4)).sizes == (9, 9, 9, 9)
    assert default_groups(g, 36) == 2


def test_generators_shapes():
    g = G.grid(5, 4)
    assert (g.num_vertices, g.num_edges) == (20, 31)
    r = G.road_like(12, 9, keep=0.2, seed=3)
    assert r.num_vertices == 108 and 107 <= r.num_edges < 12 * 8 + 11 * 9
    import oracle as O
    d, _, _, info = O.brandes_single_source(r, 0)
    assert info["reached"] == 108          # a spanning tree is inside: connected
    e = G.erdos_renyi(64, 256, seed=2)
    assert e.num_vertices == 64 and e.num_edges <= 256
    a = G.random_connected(30, 10, seed=4)
    assert O.brandes_single_source(a, 0)[3]["reached"] == 30


def test_local_rows_for_graph_partitioned_mode():
    from paper_2008_05718_b200.partitioned import local_rows
    g = G.grid(6, 5)
    part = P.strip_partition(6, 5, 3)
    total = 0
    for r in range(3):
        lg = local_rows(g, part.assignment, r)
        own = part.assignment == r
        deg = np.diff(lg.offsets)
        assert (deg[~own] == 0).all() and (deg[own] == np.diff(g.offsets)[own]).all()
        for v in np.flatnonzero(own)[:5]:
            assert lg.col_idx[lg.offsets[v]:lg.offsets[v + 1]].tolist() == \
                g.col_idx[g.offsets[v]:g.offsets[v + 1]].tolist()
        total += len(lg.col_idx)
    assert total == g.num_arcs


def test_local_graph_owned_plus_halo_numbering():
    """A rank's state arrays cover its own vertices + the other parts' borders next to them, not
    the whole graph; every rank lists all borders and its own cut arcs in local ids."""
    from paper_2008_05718_b200.partitioned import LocalGraph, incoming_cut_arcs
    for g, part in ((G.grid(8, 6), P.strip_partition(8, 6, 4)), (G.rmat(9, 6, 1), None)):
        if part is None:
            part = P.block_partition(g, 3)
        k = part.num_parts
        bs = P.identify_borders(g, part)
        a = np.asarray(part.assignment)
        covered = 0
        for r in range(k):
            lg = LocalGraph(g, part, bs, r)
            assert lg.n_local == lg.n_own + lg.n_halo + (k - 1)
            assert lg.n_own == int((a == r).sum())
            # halo = exactly the foreign endpoints of this rank's cut arcs
            src, dst = np.asarray(bs.cut_src), np.asarray(bs.cut_dst)
            want_halo = np.unique(dst[a[src] == r])
            assert sorted(lg.halo.tolist()) == want_halo.tolist()
            # rows: owned vertices keep their adjacency (mapped), the rest is empty
            deg = np.diff(lg.graph.offsets)
            assert (deg[lg.n_own:] == 0).all()
            back = np.concatenate([lg.owned, lg.halo])
            for i in range(0, lg.n_own, max(1, lg.n_own // 7)):
                v = lg.owned[i]
                mine = back[lg.graph.col_idx[lg.graph.offsets[i]:lg.graph.offsets[i + 1]]]
                assert mine.tolist() == g.col_idx[g.offsets[v]:g.offsets[v + 1]].tolist()
            # border lists: own borders are owned ids, foreign ones halo ids or the part's catch-all
            assert lg.border_off.tolist() == np.concatenate(([0], np.cumsum(bs.counts()))).tolist()
            for q in range(k):
                lv = lg.border_v[lg.border_off[q]:lg.border_off[q + 1]]
                glob = np.asarray(bs.border_arrays[q])
                if q == r:
                    assert (lv < lg.n_own).all() and (lg.owned[lv] == glob).all()
                else:
                    in_halo = np.isin(glob, lg.halo)
                    assert (back[lv[in_halo]] == glob[in_halo]).all()
                    assert (lv[~in_halo] == lg.catch_all[q]).all()
                    assert (lg.assignment[lv] == q).all()
            # own cut arcs, border by border
            mine = np.asarray(bs.border_arrays[r])
            assert len(lg.cut_off) == len(mine) + 1 and lg.cut_off[-1] == int((a[src] == r).sum())
            for j in range(0, len(mine), max(1, len(mine) // 5)):
                far = back[lg.cut_dst[lg.cut_off[j]:lg.cut_off[j + 1]]]
                assert far.tolist() == dst[src == mine[j]].tolist()
            # sources: owned or halo ids, -1 elsewhere
            loc = lg.local_of[np.arange(g.num_vertices)]
            assert ((loc >= 0) == (np.isin(np.arange(g.num_vertices), back))).all()
            covered += lg.n_own
            assert lg.n_local < g.num_vertices or k == 1 or g.num_vertices < 64
        assert covered == g.num_vertices
        cin_off, cin_src = incoming_cut_arcs(bs, bs.border_arrays)
        assert cin_off[-1] == len(bs.cut_src) == len(cin_src)


def test_reference_acceptance_corpus_host_side():
    """The reference's acceptance corpus (test_acceptance.py:69-153; digest produced by
    tests/golden/gen_acceptance_corpus.py): the generator builds the same 200 graphs, the restated
    greedy_bipartition returns the reference's assignment on every one of them, and the CPU oracle
    reproduces the reference's BC (half of the graphs are weighted)."""
    import json
    import os
    import oracle as O
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "acceptance_corpus.json")) as fh:
        doc = json.load(fh)
    assert len(doc["records"]) == 200
    for rec in doc["records"]:
        g = G.random_connected(rec["n"], rec["extra"], seed=1000 + rec["i"], weighted=rec["weighted"])
        assert g.num_edges == rec["m"] and g.unit_weight == (not rec["weighted"])
        p = P.greedy_bipartition(g, rec["ratio"], seed=rec["i"], restarts=4)
        assert "".join(str(int(x)) for x in p.assignment) == rec["assignment"], rec["i"]
        bc, _ = O.brandes_bc(g, rec["sources"], threads=1)
        assert np.allclose(bc, rec["bc"], rtol=1e-9, atol=1e-12), rec["i"]


def test_grow_partition_regions():
    """k regions grown breadth-first: valid, near-balanced on connected
    graphs, far fewer borders than id blocks once vertex ids carry no locality."""
    from paper_2008_05718_b200.partition import grow_partition
    g = G.road_like(64, 64, keep=0.2, seed=3)
    perm = np.random.default_rng(1).permutation(g.num_vertices)
    keep = g.arc_src < g.arc_dst
    gp = P.from_edge_arrays(g.num_vertices, perm[g.arc_src[keep]], perm[g.arc_dst[keep]])
    for k in (2, 3, 8):
        p = grow_partition(gp, k, seed=0)
        sizes = np.bincount(p.assignment, minlength=k)
        assert p.num_parts == k and len(p.assignment) == gp.num_vertices
        assert sizes.min() > 0 and sizes.max() <= 1.6 * gp.num_vertices / k
        grown = sum(P.identify_borders(gp, p).counts())
        blocks = sum(P.identify_borders(gp, P.block_partition(gp, k)).counts())
        assert grown * 5 < blocks
        assert np.array_equal(p.assignment, grow_partition(gp, k, seed=0).assignment)      # deterministic
    # disconnected graph with isolated vertices: every vertex gets a part
    h = P.from_edge_arrays(300, list(range(0, 99)) + list(range(150, 249)), list(range(1, 100)) + list(range(151, 250)))
    for k in (2, 5):
        a = grow_partition(h, k, seed=2).assignment
        assert a.min() >= 0 and a.max() < k
    assert make_partition(gp, P.RunConfig(num_partitions=4, partitioner="grow")).num_parts == 4
    with pytest.raises(P.InputError):
        P.RunConfig(partitioner="metis")


def test_bench_reference_arm_line_shape():
    """`bench.py --impl reference` runs on the host cores only (the CPU oracle port) and prints the
    contract's JSON line; smoke-size workload so the CPU suite stays fast."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--workload", "rmat16",
                          "--sources", "32", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-500:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "bc_teps" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    for key in ("unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "config"):
        assert key in line


def test_import_partition_file(tmp_path):
    """METIS-style partition files (reference partition.py:112-136; test_engine.py:118-123)."""
    g = G.path(6)
    f = tmp_path / "p.txt"
    f.write_text("0\n0\n\n1\n1\n2\n2\n")           # blank lines are skipped
    p = P.import_partition(str(f), g, 3)
    assert p.assignment.tolist() == [0, 0, 1, 1, 2, 2] and p.num_parts == 3
    assert abs(p.ratio - 2 / 6) < 1e-12
    bs = P.identify_borders(g, p)
    assert [b.tolist() for b in bs.border_arrays] == [[1], [2, 3], [4]]
    f.write_text("0\n1\nx\n")
    with pytest.raises(P.FormatError, match="line 3"):
        P.import_partition(str(f), g, 2)
    f.write_text("0\n1\n2\n0\n0\n0\n")
    with pytest.raises(P.FormatError, match="outside"):
        P.import_partition(str(f), g, 2)
    f.write_text("0\n1\n")
    with pytest.raises(P.FormatError, match="2 lines"):
        P.import_partition(str(f), g, 2)
    f.write_text("0\n" * 6)
    with pytest.warns(UserWarning, match="empty"):
        assert P.import_partition(str(f), g, 2).degenerate
    # through the front door: partition_file feeds make_partition
    from paper_2008_05718_b200.engine import make_partition
    f.write_text("0\n0\n0\n1\n1\n1\n")
    cfg = P.RunConfig(partition_file=str(f), num_partitions=2)
    assert make_partition(g, cfg).assignment.tolist() == [0, 0, 0, 1, 1, 1]


def test_mode_falls_back_when_the_border_tables_do_not_fit():
    """hybir needs b_p^2 x 12 B of tables per part; above the budget run_bc switches to the
    reference's other partitioned mode instead of failing (SURVEY.md hard part 2)."""
    g = G.rmat(10, 8, 1)
    bs = P.identify_borders(g, P.block_partition(g, 2))
    need = P.border_table_bytes(bs)
    assert need == sum(12.0 * b * b for b in bs.counts()) and need > 0
    assert P.choose_mode("hybir", bs, need) == "hybir"
    with pytest.warns(UserWarning, match="bsp-baseline"):
        assert P.choose_mode("hybir", bs, need - 1) == "bsp-baseline"
    assert P.choose_mode("bsp-baseline", bs, 0) == "bsp-baseline"
    assert P.choose_mode("direct", bs, 0) == "direct"


def test_load_dimacs_gr(tmp_path):
    f = tmp_path / "g.gr"
    f.write_text("c comment\np sp 4 4\na 1 2 3\na 2 1 3\na 2 3 1\na 4 3 2\n")
    g = P.load_dimacs_gr(str(f))
    assert (g.num_vertices, g.num_edges) == (4, 3)
    assert g.offsets.tolist() == [0, 1, 3, 5, 6]
    assert g.arc_weight.tolist() == [3, 3, 1, 1, 2, 2]
    f.write_text("p sp 2 2\na 1 2 1\n")
    with pytest.raises(P.FormatError, match="declares 2 arcs"):
        P.load_dimacs_gr(str(f))
    f.write_text("a 1 2 1\n")
    with pytest.raises(P.ParseError):
        P.load_dimacs_gr(str(f))
    f.write_text("p sp 2 1\na 1 3 1\n")
    with pytest.raises(P.FormatError, match="out of range"):
        P.load_dimacs_gr(str(f))


def test_refine_partition_lowers_the_cut_and_keeps_the_balance():
    from paper_2008_05718_b200.partition import cut_size
    for g, k in ((G.road_like(96, 96, keep=0.2, seed=3), 4), (G.grid(40, 40), 3), (G.rmat(11, 8, 2), 4)):
        n = g.num_vertices
        for start in (P.block_partition(g, k), P.grow_partition(g, k, seed=1)):
            out = P.refine_partition(g, start)
            assert out.num_parts == k and len(out.assignment) == n
            assert cut_size(g, out) <= cut_size(g, start)
            assert max(out.sizes) <= int(1.05 * n / k) + 1 or max(out.sizes) <= max(start.sizes)
        best = P.mincut_partition(g, k, seed=0)
        assert cut_size(g, best) <= cut_size(g, P.grow_partition(g, k, seed=0))
    # a scrambled grid: refinement must recover most of the locality
    g = G.grid(32, 32)
    rng = np.random.default_rng(0)
    noisy = P.strip_partition(32, 32, 2).assignment.copy()
    flip = rng.random(len(noisy)) < 0.1
    noisy[flip] = 1 - noisy[flip]
    start = P.Partition(noisy, 0.5, 2)
    assert cut_size(g, P.refine_partition(g, start)) < cut_size(g, start) // 2


def test_grown_partitions_stay_balanced_on_trees():
    """Regions that fill up seal subtrees off; the leftovers are dealt out by room, not flooded into
    the neighbouring (full) part."""
    g = G.random_connected(20000, 150, seed=3)
    for k in (2, 4, 8):
        for p in (P.grow_partition(g, k, seed=0), P.mincut_partition(g, k, seed=0)):
            sizes = np.asarray(p.sizes)
            assert sizes.sum() == g.num_vertices and sizes.min() > 0
            assert sizes.max() <= 1.12 * g.num_vertices / k, (k, p.sizes)


def test_bench_samples_are_strided():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    srcs = list(range(0, 2048, 2))
    s = bench.strided_sample(srcs, 16)
    assert len(s) == 16 and s[0] == srcs[0] and s == sorted(set(s))
    assert max(np.diff(s)) == min(np.diff(s)) == 128           # evenly spread, not a prefix
    assert bench.strided_sample(srcs, 5000) == srcs
    g = G.rmat(12, 8, 1)
    all_src = bench.pick_sources(g.num_vertices, 1024)
    full = bench.isolated_fraction(g, all_src)
    assert abs(bench.isolated_fraction(g, bench.strided_sample(all_src, 256)) - full) < 0.08

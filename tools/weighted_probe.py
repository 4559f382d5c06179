"""General-weight sweeps at size (dev tool, GPU box): road-like grid with DIMACS-style weights,
timing of bc_run and a parity sample against the C oracle's Dijkstra."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine

side = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n_src = int(sys.argv[2]) if len(sys.argv) > 2 else 128
wmax = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
base = G.road_like(side, side, seed=1)
rng = np.random.default_rng(5)
src, dst = base.arc_src, base.arc_dst
keep = src < dst
g = P.from_edge_arrays(base.num_vertices, src[keep], dst[keep], rng.integers(1, wmax + 1, size=int(keep.sum())))
srcs = sorted(np.random.default_rng(2).choice(g.num_vertices, n_src, replace=False).tolist())
print("n", g.num_vertices, "m", g.num_edges, "sources", n_src, "wmax", int(g.arc_weight.max()), flush=True)
with Engine(g) as e:
    e.set_option("groups", max(1, min(16, n_src // 32)))
    if os.environ.get("SSSP_BLOCKS"):
        e.set_option("sssp_blocks", int(os.environ["SSSP_BLOCKS"]))
    if os.environ.get("SSSP_DELTA"):
        e.set_option("sssp_delta", int(os.environ["SSSP_DELTA"]))
    e.run(srcs[:32])
    t0 = time.perf_counter()
    bc, st = e.run(srcs)
    dt = time.perf_counter() - t0
    print("bc_run %.1f ms  (%.2f MTEPS)  DAG depth %d  launches %d  fwd %.1f ms  bwd %.1f ms" % (
        dt * 1e3, g.num_edges * n_src / dt / 1e6, st["max_levels"], st["launches"], st["ms_forward"], st["ms_backward"]), flush=True)
    sample = srcs[:: max(1, n_src // 8)][:8]
    t0 = time.perf_counter()
    obc, info = O.brandes_bc(g, sample)
    t_cpu = time.perf_counter() - t0
    gbc, _ = e.run(sample)
    print("oracle %d sources %.2f s (%.2f MTEPS); parity %s" % (
        len(sample), t_cpu, g.num_edges * len(sample) / t_cpu / 1e6, bool(np.allclose(gbc, obc, rtol=1e-9, atol=1e-12))), flush=True)

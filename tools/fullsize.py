"""Record runs of the full-size BASELINE configurations on one B200 (dev tool)."""
import json, os, random, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_DIRECT, MODE_HYBIR, MODE_BSP

def log(**kw):
    print(json.dumps(kw), flush=True)

def run_direct(name, g, nsrc, groups, check=16, seed=0, relabel=-1):
    srcs = sorted(random.Random(seed).sample(range(g.num_vertices), nsrc))
    with Engine(g) as e:
        e.set_option("groups", groups)
        if relabel >= 0:
            e.set_option("relabel", relabel)
        e.run(srcs)            # warm-up: state, level arrays and queues at their final sizes
        t0 = time.time(); bc, st = e.run(srcs); wall = time.time() - t0
        bcs, _ = e.run(srcs[:check])
    t0 = time.time(); obc, info = O.brandes_bc(g, srcs[:check]); cpu = time.time() - t0
    rel = float(np.max(np.abs(bcs - obc) / np.maximum(np.abs(obc), 1e-9)))
    fwd = 8 * st["arcs_reached"] + 16 * st["dag_arcs"] + 28 * st["reached"]
    bwd = 8 * st["arcs_reached"] + 16 * st["dag_arcs"] + 44 * st["reached"]
    log(config=name, n=g.num_vertices, m=g.num_edges, sources=nsrc, groups=groups, ms=st["ms_total"], wall_s=wall,
        gteps=g.num_edges * nsrc / st["ms_total"] / 1e6, fwd_ms=st["ms_forward"], bwd_ms=st["ms_backward"],
        levels=st["max_levels"], launches=st["launches"], alg_GBps=(fwd + bwd) / st["ms_total"] / 1e6,
        bc_rel_vs_oracle=rel, oracle_sigma_max=info["sigma_max"], cpu_teps=g.num_edges * check / cpu, cpu_threads=info["threads"])

which = sys.argv[1:] or ["c1", "rmat22", "er22", "road2048", "grid512_hybir"]
if "rmat22" in which:
    t = time.time(); g = G.rmat(22, 16, 1); log(built="rmat22", s=time.time() - t)
    run_direct("R-MAT s22 ef16, 4096 sources (north-star target)", g, 4096, 8)
    del g
if "er22" in which:
    t = time.time(); g = G.erdos_renyi(1 << 22, 1 << 26, 1); log(built="er22", s=time.time() - t)
    run_direct("Erdos-Renyi 4M deg 32, 4096 sources (config 4, one GPU's view)", g, 4096, 8)
    del g
if "road2048" in which:
    t = time.time(); g = G.road_like(2048, 2048, keep=0.2, seed=1); log(built="road2048", s=time.time() - t)
    run_direct("road-like 2048x2048, 512 sources (config 3 graph, unpartitioned)", g, 512, 4, check=8)
    run_direct("road-like 2048x2048, 512 sources, one batch of 16 groups", g, 512, 16, check=8)
    del g
if "grid512_hybir" in which:
    g = G.road_like(512, 512, keep=0.2, seed=1)
    for k in (2, 4, 8):
        part = P.strip_partition(512, 512, k)
        srcs = sorted(random.Random(0).sample(range(g.num_vertices), 128))
        with Engine(g) as e:
            e.set_option("groups", 4); e.set_option("reports", 0)
            t0 = time.time(); e.set_partition(k, part.assignment); counts = e.border_counts(k).tolist()
            bc, st = e.run(srcs, MODE_HYBIR); wall = time.time() - t0
            bcd, std = e.run(srcs, MODE_DIRECT)
        obc, info = O.brandes_bc(g, srcs[:16])
        with Engine(g) as e:
            e.set_option("reports", 0); e.set_partition(k, part.assignment)
            b16, _ = e.run(srcs[:16], MODE_HYBIR)
        log(config="road-like 512x512 hybir, %d strips" % k, borders=counts, sources=128, ms=st["ms_total"], ms_border=st["ms_border"],
            wall_incl_tables_s=wall, iterations=st["iterations"], levels=st["max_levels"], direct_ms=std["ms_total"],
            hybir_vs_direct=float(np.max(np.abs(bc - bcd) / np.maximum(np.abs(bcd), 1e-9))),
            bc_rel_vs_oracle=float(np.max(np.abs(b16 - obc) / np.maximum(np.abs(obc), 1e-9))), sigma_max=info["sigma_max"])
if "c1" in which:
    # BASELINE config 1: R-MAT s12 ef8, ALL sources, 2 partitions (the reference's own partitioner)
    g = G.rmat(12, 8, 1)
    srcs = list(range(g.num_vertices))
    t0 = time.time(); obc, info = O.brandes_bc(g, srcs); cpu = time.time() - t0
    for mode in ("direct", "bsp-baseline", "hybir"):
        P.run_bc(g, P.RunConfig(sources=srcs, mode=mode, num_partitions=2, per_source_reports=True))   # warm-up at full size
        t0 = time.time()
        res = P.run_bc(g, P.RunConfig(sources=srcs, mode=mode, num_partitions=2, per_source_reports=True))
        wall = time.time() - t0
        log(config="config 1: R-MAT s12 ef8, all 4096 sources, 2 parts, mode=%s" % mode, n=g.num_vertices, m=g.num_edges,
            borders=list(res.borders.counts()), wall_s=wall, device_ms=res.stats["ms_total"], border_ms=res.stats["ms_border"],
            mteps_e2e=res.mteps, bc_rel_vs_oracle=float(np.max(np.abs(res.bc - obc) / np.maximum(np.abs(obc), 1e-9))),
            iterations=res.stats["iterations"], comm_events=res.stats["comm_events"], sync_events=res.stats["sync_events"],
            cpu_port_s=cpu, cpu_threads=info["threads"])
if "rmat24" in which:
    # BASELINE config 5 graph on ONE GPU (the configuration itself is an 8-GPU run)
    t = time.time(); g = G.rmat(24, 16, 1); log(built="rmat24", s=time.time() - t, n=g.num_vertices, m=g.num_edges)
    # (a sample of a 4096-source job: renumbered as that job would be after its first 2048 sources)
    run_direct("R-MAT s24 ef16, 256 of the 4096 sources, one GPU, renumbered ids", g, 256, 4, check=4, relabel=1)
    del g
if "road2048_hybir" in which:
    # BASELINE config 3 on ONE GPU: the k strips that would sit on k GPUs run in one address space
    g = G.road_like(2048, 2048, keep=0.2, seed=1)
    # Step 1 / Step 6 / the border-table searches run on frontier queues (no dense level rows), so
    # all 512 sources of config 3 go in one batch of 16 groups
    nsrc, groups = 512, 16
    srcs = sorted(random.Random(0).sample(range(g.num_vertices), nsrc))
    for k in (8, 2):
        part = P.strip_partition(2048, 2048, k)
        with Engine(g) as e:
            e.set_option("groups", groups); e.set_option("reports", 0)
            t0 = time.time(); e.set_partition(k, part.assignment); counts = e.border_counts(k).tolist()
            t1 = time.time(); bc, st = e.run(srcs[:32], MODE_HYBIR); t_tables = time.time() - t1   # builds the tables
            t2 = time.time(); bc, st = e.run(srcs, MODE_HYBIR); wall = time.time() - t2
            bcd, std = e.run(srcs, MODE_DIRECT)
        log(config="road-like 2048x2048 hybir (queue sweeps), %d strips, %d sources, groups=%d" % (k, nsrc, groups),
            borders=counts, ms=st["ms_total"],
            ms_border=st["ms_border"], ms_forward=st["ms_forward"], ms_backward=st["ms_backward"], wall_s=wall,
            set_partition_s=t1 - t0, tables_and_first_batch_s=t_tables, iterations=st["iterations"],
            levels=st["max_levels"], launches=st["launches"], direct_ms=std["ms_total"],
            gteps=g.num_edges * nsrc / st["ms_total"] / 1e6,
            hybir_vs_direct=float(np.max(np.abs(bc - bcd) / np.maximum(np.abs(bcd), 1e-9))))

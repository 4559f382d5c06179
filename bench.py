#!/usr/bin/env python
"""Benchmark of the BC hot path: BC TEPS = sources x edges / second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload at N = 1: BASELINE.json configs[1] -- R-MAT scale-20, edge factor 16,
1024 sampled sources (``sorted(random.Random(0).sample(range(n), 1024))``, the
reference's sampling rule, engine.py:82-84), one B200.  A *step* is one full
BC computation over that source list.  At N > 1 (launched by torchrun, one
rank per GPU) the graph is replicated and every rank adds 1024 more sources
(weak scaling, source-sharded mode); the single all-reduce of the BC vector
is inside the timed region.

Printed JSON (one line, rank 0):
  value     whole-job TEPS, graph resident in HBM, timed with CUDA events on
            the stream the kernels run on, max over ranks
  e2e       same metric through the public call ``run_bc(g, cfg)`` with host
            buffers: CSR + sources host->device, BC vector device->host, inside
            the timed region (wall clock bracketed by device synchronisation)
  roofline  level kernels (forward + backward sweeps): algorithmic bytes
             / device time against the measured HBM copy bandwidth
  cpu_baseline  the C/OpenMP oracle port of the reference's sequential Brandes
            on the box's host cores, bounded source sample
``--impl reference`` times that CPU port alone (the reference itself is
pure Python and single-threaded; the port is bit-identical to it, see
tests/test_oracle.py) and prints the same line shape with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "bc_teps"
UNIT = "TEPS (sources*edges/s)"


def workload(name: str):
    from paper_2008_05718_b200 import generators as G
    if name == "rmat20":
        g = G.rmat(20, 16, 1)
        label = "R-MAT scale-20 edge-factor-16 (a,b,c)=(.57,.19,.19) seed 1, undirected unweighted"
    elif name == "rmat22":
        g = G.rmat(22, 16, 1)
        label = "R-MAT scale-22 edge-factor-16 (a,b,c)=(.57,.19,.19) seed 1, undirected unweighted"
    elif name == "rmat16":
        g = G.rmat(16, 16, 1)
        label = "R-MAT scale-16 edge-factor-16 (smoke-size)"
    elif name == "road2048":
        g = G.road_like(2048, 2048, keep=0.2, seed=1)
        label = "road-like 2048x2048 (random spanning tree of the grid + 20% of the other grid edges)"
    elif name == "road512":
        g = G.road_like(512, 512, keep=0.2, seed=1)
        label = "road-like 512x512 (smoke-size)"
    elif name == "er22":
        g = G.erdos_renyi(1 << 22, 1 << 26, 1)
        label = "Erdos-Renyi n=2^22, 2^26 random pairs (avg degree 32)"
    else:
        raise SystemExit("unknown workload %r" % name)
    return g, label


def pick_sources(n: int, k: int, seed: int = 0):
    return sorted(random.Random(seed).sample(range(n), min(k, n)))


def measured_peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.proc = None
        self.path = None
        self.index = device_index

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
            os.unlink(self.path)
        except Exception:
            return out
        sm, reasons = [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                out["sm_max_mhz"] = float(r[2])
            except ValueError:
                continue
            for name, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if sm:
            # "under load" = the upper half of the samples (idle clocks sit low)
            sm.sort()
            out["sm_mhz"] = statistics.median(sm[len(sm) // 2:])
            out["samples"] = len(sm)
        out["reasons"] = sorted(reasons)
        return out


def ncu_traffic(workload_name: str):
    """DRAM bytes the level kernel moved per launch (mean over the forward and backward
    launches of one batch), from the committed ncu `--set full` capture
    (profiles/r1_traffic.json, written by tools/summarize_profiles.py; null when no capture matches)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as fh:
            rec = json.load(fh)
        return rec.get(workload_name)
    except Exception:
        return None


def algorithmic_bytes(st: dict, n: int):
    """forward 8*A_r + 16*T + 28*n_r, backward 8*A_r + 16*T + 44*n_r,
    initialisation 20*n per source."""
    fwd = 8 * st["arcs_reached"] + 16 * st["dag_arcs"] + 28 * st["reached"]
    bwd = 8 * st["arcs_reached"] + 16 * st["dag_arcs"] + 44 * st["reached"]
    init = 20 * n * st["sources"]
    return fwd, bwd, init


def cpu_sample(g, sources, seconds_target=15.0):
    """Time the oracle port on a bounded prefix of the source list."""
    import oracle as O
    threads = O.host_threads()
    k = min(len(sources), max(threads, 2 * threads))
    t0 = time.perf_counter()
    O.brandes_bc(g, sources[:k], threads=threads)
    dt = time.perf_counter() - t0
    # one refinement so the sample lands near the target duration
    if dt < seconds_target / 3 and k < len(sources):
        k2 = min(len(sources), int(k * min(64.0, seconds_target / max(dt, 1e-3))))
        k2 = max(threads, (k2 // threads) * threads)
        if k2 > k:
            k = k2
            t0 = time.perf_counter()
            O.brandes_bc(g, sources[:k], threads=threads)
            dt = time.perf_counter() - t0
    return {"value": g.num_edges * k / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "first %d of the %d sources, %.1f s on %d OpenMP threads (oracle/brandes_oracle.c)"
                      % (k, len(sources), dt, threads)}, k, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    g, label = workload(args.workload)
    sources = pick_sources(g.num_vertices, args.sources)
    import oracle as O
    threads = O.host_threads()
    # bounded sample per step: sized from one probe so W + K steps end within minutes
    probe, k, dt = cpu_sample(g, sources, seconds_target=8.0)
    per_source = dt / k
    budget = 150.0 / max(1, args.steps + args.warmup)
    k_step = int(min(len(sources), max(threads, budget / per_source)))
    k_step = max(threads, (k_step // threads) * threads)
    for _ in range(args.warmup):
        O.brandes_bc(g, sources[:k_step], threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.brandes_bc(g, sources[:k_step], threads=threads)
    dt = time.perf_counter() - t0
    value = g.num_edges * k_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": label, "n": g.num_vertices, "m": g.num_edges,
                   "sources": len(sources), "sources_per_step": k_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "%d of the %d sources per step on %d OpenMP threads; the reference "
                                   "is pure Python (1 core), this is its bit-identical C restatement"
                                   % (k_step, len(sources), threads)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_partitioned(args):
    """--gpu-mode graph-partitioned: one part per rank, strong scaling (all ranks work on the same
    sources).  Forward phase per --forward: hybir = border matrices (two all-reduces per batch),
    bsp = one border exchange per level.  Not the default line; for the multi-GPU record runs."""
    import torch
    import torch.distributed as dist

    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200.multigpu import init_process_group
    from paper_2008_05718_b200.partitioned import PartitionedRunner

    rank, world = init_process_group("nccl")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    g, label = workload(args.workload)
    n, m = g.num_vertices, g.num_edges
    sources = pick_sources(n, args.sources)
    if args.workload.startswith("road"):
        side = int(args.workload[4:])
        part = P.strip_partition(side, side, world)
    elif args.partitioner == "grow":
        part = P.grow_partition(g, world, seed=0)
    else:
        part = P.block_partition(g, world)
    runner = PartitionedRunner(g, part, dev, args.groups or 4, args.forward)
    for _ in range(args.warmup):
        runner.run(sources)
    dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        bc = runner.run(sources)
    ev1.record()
    dist.barrier()
    torch.cuda.synchronize(dev)
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    line = {
        "metric": METRIC, "value": m * len(sources) * args.steps / (float(ms.item()) / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(ms.item()) / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "n": n, "m": m, "sources": len(sources), "mode": "graph-partitioned",
                   "forward": args.forward, "borders": runner.border_counts, "levels": runner.levels,
                   "forward_exchanges_per_step": runner.forward_exchanges / max(1, args.steps + args.warmup),
                   "backward_exchanges_per_step": runner.backward_exchanges / max(1, args.steps + args.warmup),
                   "exchanged_bytes_per_step": runner.exchanged_bytes / max(1, args.steps + args.warmup)},
        "bc_sum": float(bc.sum().item()),
    }
    runner.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200._capi import Engine, MODE_DIRECT
    from paper_2008_05718_b200.engine import default_groups

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # launched by torchrun (even with one rank): join the NCCL job, so the N = 1 line of a scaling
    # run goes through the same collectives as N > 1
    use_dist = world > 1 or ("RANK" in os.environ and "MASTER_ADDR" in os.environ)
    if use_dist:
        from paper_2008_05718_b200.multigpu import init_process_group
        init_process_group("nccl")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the engine has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    g, label = workload(args.workload)
    g.pin()                                    # e2e copies the CSR from pinned host memory
    n, m = g.num_vertices, g.num_edges
    all_sources = pick_sources(n, args.sources * world)
    mine = all_sources[rank::world]            # 1024 per rank: weak scaling
    groups = args.groups or default_groups(g, len(mine))

    eng = Engine(g, local)
    eng.set_option("groups", groups)
    if args.item_arcs:
        eng.set_option("item_arcs", args.item_arcs)
    bc_dev = torch.zeros(n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        bc_dev.zero_()
        st = eng.run_device(mine, bc_dev.data_ptr(), stream.cuda_stream, MODE_DIRECT)
        if use_dist:
            dist.all_reduce(bc_dev, op=dist.ReduceOp.SUM)
        return st

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        st = step()
    sampler = ClockSampler(local)
    barrier()
    if rank == 0:
        sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    acc = {"ms_forward": 0.0, "ms_backward": 0.0, "launches": 0, "launches_forward": 0, "launches_backward": 0,
           "launches_level": 0, "ms_level": 0.0, "launches_level_timed": 0}
    ev0.record(stream)
    for _ in range(args.steps):
        st = step()
        for key in acc:
            acc[key] += st[key]
    ev1.record(stream)
    barrier()
    clocks = sampler.stop() if rank == 0 else {}
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_total = float(ms.item())
    value = m * len(all_sources) * args.steps / (ms_total / 1e3)

    # ---- end to end through the public API: host CSR in, host BC vector out
    eng.close()
    cfg = P.RunConfig(sources=mine, mode="direct", device=local, groups=groups,
                      item_arcs=args.item_arcs or None, per_source_reports=False)
    e2e_steps = max(1, min(args.steps, 3))
    P.run_bc(g, cfg)                       # warm-up (allocator, page-in)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = P.run_bc(g, cfg)
        if use_dist:
            t = torch.from_numpy(res.bc).to(dev)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            res.bc[:] = t.cpu().numpy()
    barrier()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = m * len(all_sources) * e2e_steps / float(e2e_s.item())
    h2d = g.offsets.nbytes + g.col_idx.nbytes + 8 * len(mine)
    d2h = 8 * n + 64
    if use_dist:   # the host BC vector goes back to the device for the all-reduce and returns
        h2d += 8 * n
        d2h += 8 * n

    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    peak, peak_src = measured_peak_gbs()
    fwd_b, bwd_b, init_b = algorithmic_bytes(st, n)
    fwd_ms = acc["ms_forward"] / args.steps
    bwd_ms = acc["ms_backward"] / args.steps
    lf = acc["launches_forward"] / args.steps
    lb = acc["launches_backward"] / args.steps

    def sweep(nbytes, ms, launches):
        gbs = nbytes / (ms / 1e3) / 1e9
        return {"achieved": gbs, "frac": gbs / peak, "algorithmic_bytes_per_step": nbytes, "ms_per_step": ms,
                "launches_per_step": launches, "bytes_per_launch": nbytes / max(launches, 1),
                "avg_launch_ms": ms / max(launches, 1)}

    both = sweep(fwd_b + bwd_b, fwd_ms + bwd_ms, lf + lb)
    # the dominant kernel alone: CUDA events around every level-kernel launch (bc_stats.ms_level)
    traffic = ncu_traffic(args.workload)
    lvl_ms = acc["ms_level"] / args.steps
    lvl_n = acc["launches_level_timed"] / args.steps
    lvl_avg = lvl_ms / max(lvl_n, 1)
    level_kernel = {
        "ms_per_step": lvl_ms, "launches_per_step": lvl_n, "avg_launch_ms": lvl_avg,
        "share_of_step": lvl_ms / (ms_total / args.steps),
        "algorithmic_bytes_per_launch": (fwd_b + bwd_b) / max(lvl_n, 1),
        "algorithmic_achieved": (fwd_b + bwd_b) / max(lvl_ms, 1e-9) / 1e6,
        "dram_bytes_per_launch": traffic,
        "dram_achieved": (traffic / (lvl_avg / 1e3) / 1e9) if traffic and lvl_avg > 0 else None,
        "dram_frac": (traffic / (lvl_avg / 1e3) / 1e9 / peak) if traffic and lvl_avg > 0 else None,
        "note": "dram_* = DRAM bytes per launch from the committed ncu --set full capture (roofline.traffic) "
                "over the live average launch time: what the kernel really pulls from HBM",
    }
    roofline = {
        "bound": "hbm", "kernel": "level_kernel<forward | backward> and the push / queue kernels of the same sweeps",
        "achieved": both["achieved"], "peak": peak, "unit": "GB/s", "frac": both["frac"],
        "traffic": traffic, "peak_source": peak_src,
        "algorithmic_bytes_per_step": both["algorithmic_bytes_per_step"], "ms_per_step": both["ms_per_step"],
        "launches_per_step": both["launches_per_step"], "bytes_per_launch": both["bytes_per_launch"],
        "avg_launch_ms": both["avg_launch_ms"],
        "level_kernel_launches_per_step": acc["launches_level"] / args.steps,
        "algorithmic_bytes_per_level_kernel_launch": (fwd_b + bwd_b) / max(1.0, acc["launches_level"] / args.steps),
        "level_kernel": level_kernel,
        "forward": sweep(fwd_b, fwd_ms, lf), "backward": sweep(bwd_b, bwd_ms, lb),
        "whole_step": {"achieved": (fwd_b + bwd_b + init_b) / (ms_total / args.steps / 1e3) / 1e9,
                       "frac": (fwd_b + bwd_b + init_b) / (ms_total / args.steps / 1e3) / 1e9 / peak},
        "note": "algorithmic bytes count every source separately (SURVEY.md 8d); 32 sources share one "
                "adjacency read and most sigma rows are served by L2, so frac > 1 is expected and the "
                "kernel is latency / L1-throughput bound (profiles/)",
    }
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu, _, _ = cpu_sample(g, all_sources)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "n": n, "m": m, "sources": len(all_sources),
                   "sources_per_gpu": len(mine), "mode": "source-sharded" if world > 1 else "single-gpu",
                   "groups": groups, "max_levels": st["max_levels"],
                   "l2": "per-batch state %.1f GB >> 126 MB L2, no flush needed"
                         % (groups * n * 560 / 1e9)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "call": "run_bc(g, RunConfig(sources=..., mode='direct'))"},
        "gpu_launches": int(acc["launches"]),
        "clocks": clocks,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "traversal": {k: st[k] for k in ("reached", "arcs_reached", "dag_arcs")},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="rmat20")
    ap.add_argument("--sources", type=int, default=1024, help="sources per GPU")
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--item-arcs", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--gpu-mode", default="source-sharded", choices=("source-sharded", "graph-partitioned"))
    ap.add_argument("--forward", default="hybir", choices=("hybir", "bsp"),
                    help="forward phase of the graph-partitioned mode")
    ap.add_argument("--partitioner", default="block", choices=("block", "grow"))
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpu_mode == "graph-partitioned":
        return run_partitioned(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

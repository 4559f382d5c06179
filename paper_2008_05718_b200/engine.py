"""``run_bc`` -- the reference's public BC entry point on the B200 engine.

Same call shape as the reference (reference pkg/src/hybir/engine.py:38-153):
``run_bc(g, cfg) -> RunResult`` with ``RunConfig`` carrying the reference's
fields (``num_sources, sources, seed, ratio, mode, backward_strategies,
partition_file, calibration_sources, max_threads``) plus the new ones the
north star names: ``num_partitions`` (the reference is fixed at two),
``num_gpus`` / ``gpu_mode`` for the one-process-per-GPU multi-GPU modes, and
tuning knobs.  The host code here does source selection, partitioning, border
identification and source batching; every arithmetic step runs in the CUDA
library behind ``_capi.Engine``.
"""

from __future__ import annotations

import hashlib
import os
import random
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .errors import InputError
from .graph import Graph, graph_stats
from .partition import (BorderSet, Partition, block_partition, greedy_bipartition, grow_partition,
                        identify_borders, import_partition, mincut_partition, single_partition)

MODES = ("hybir", "bsp-baseline", "direct")
GPU_MODES = ("source-sharded", "graph-partitioned")
STRATEGIES = ("vertex-pull", "edge-push")
_MODE_CODE = {"direct": _capi.MODE_DIRECT, "hybir": _capi.MODE_HYBIR,
              "bsp-baseline": _capi.MODE_BSP}


def validate_strategy(name: str) -> str:
    if name not in STRATEGIES:
        raise InputError("unknown backward strategy %r; pick from %s" % (name, STRATEGIES))
    return name


@dataclass
class RunConfig:
    # -- reference fields (engine.py:39-47) --------------------------------
    num_sources: int | None = None     # None with sources=None means all vertices
    sources: list | None = None
    seed: int = 0
    ratio: float | str = 0.5
    mode: str = "hybir"
    backward_strategies: tuple = ("vertex-pull", "edge-push")  # accepted; the GPU pulls on every part
    partition_file: str | None = None
    calibration_sources: int = 10      # accepted; every part is an identical B200
    max_threads: int | None = None     # metadata only, as in the reference
    # -- new -------------------------------------------------------------------
    num_partitions: int = 2            # the reference's fixed value
    partition: Partition | None = None  # explicit assignment (tests, grid strips)
    partitioner: str = "auto"          # "auto": the reference's grower for 2 parts, id blocks above;
                                       # "grow": k regions grown breadth-first (grow_partition); "block";
                                       # "mincut": grown regions + boundary refinement (mincut_partition)
    table_budget_bytes: float = 64e9   # border tables above this size: hybir falls back to bsp-baseline
    table_cache_dir: str | None = None  # border-table disk cache (border_matrix.py:85-125)
    shard_border_tables: bool = True   # graph-partitioned hybir: one border table per rank (False: all on all)
    num_gpus: int = 1
    gpu_mode: str = "source-sharded"
    device: int | None = None          # CUDA ordinal; default LOCAL_RANK or 0
    groups: int | None = None          # 32-lane source groups per batch (None = heuristic)
    item_arcs: int | None = None
    per_source_reports: bool = True

    def __post_init__(self):
        if self.mode not in MODES:
            raise InputError("unknown mode %r; pick from %s" % (self.mode, MODES))
        for name in self.backward_strategies:
            validate_strategy(name)
        if self.num_sources is not None and self.num_sources < 1:
            raise InputError("num_sources must be >= 1")
        if self.num_partitions < 1:
            raise InputError("num_partitions must be >= 1")
        if self.partitioner not in ("auto", "grow", "block", "mincut"):
            raise InputError("unknown partitioner %r; pick from auto, grow, block, mincut" % self.partitioner)
        if self.gpu_mode not in GPU_MODES:
            raise InputError("unknown gpu_mode %r; pick from %s" % (self.gpu_mode, GPU_MODES))
        if self.max_threads is None and os.environ.get("HYBIR_THREADS"):
            self.max_threads = int(os.environ["HYBIR_THREADS"])


class CommTotals:
    """Cheap stand-in for the reference's ledger (ledger.py:25-59): totals only."""

    def __init__(self, forward_events=0, backward_events=0, payload_bytes=0):
        self.forward_events = int(forward_events)
        self.backward_events = int(backward_events)
        self.payload_bytes = int(payload_bytes)

    def count(self, phase=None, source=None) -> int:
        if phase == "forward":
            return self.forward_events
        if phase == "backward":
            return self.backward_events
        return self.forward_events + self.backward_events

    def totals(self) -> dict:
        return {
            "events": self.forward_events + self.backward_events,
            "forward_events": self.forward_events,
            "backward_events": self.backward_events,
            "payload_bytes": self.payload_bytes,
        }


@dataclass
class RunResult:
    bc: np.ndarray
    per_source: list
    ledger: CommTotals
    mteps: float
    elapsed: float
    partition: Partition
    borders: BorderSet
    config: RunConfig
    pipeline_overlaps: int = 0
    stats: dict = field(default_factory=dict)   # device-side timings and traversal counters


def select_sources(g: Graph, cfg: RunConfig) -> list:
    """Explicit list as given | all vertices | sorted seeded sample (engine.py:73-84)."""
    n = g.num_vertices
    if cfg.sources is not None:
        for s in cfg.sources:
            if not 0 <= s < n:
                raise InputError("listed source %d out of range [0, %d)" % (s, n))
        return list(cfg.sources)
    if cfg.num_sources is None:
        return list(range(n))
    rng = random.Random(cfg.seed)
    return sorted(rng.sample(range(n), min(cfg.num_sources, n)))


def make_partition(g: Graph, cfg: RunConfig) -> Partition:
    if cfg.partition is not None:
        if len(cfg.partition.assignment) != g.num_vertices:
            raise InputError("partition length does not match the graph")
        return cfg.partition
    if cfg.num_partitions == 1 or cfg.mode == "direct":
        return single_partition(g)
    if cfg.partition_file is not None:
        return import_partition(cfg.partition_file, g, cfg.num_partitions)
    if cfg.partitioner == "grow":
        return grow_partition(g, cfg.num_partitions, seed=cfg.seed)
    if cfg.partitioner == "block":
        return block_partition(g, cfg.num_partitions)
    if cfg.partitioner == "mincut":
        return mincut_partition(g, cfg.num_partitions, seed=cfg.seed)
    if cfg.num_partitions == 2:
        # 'auto' calibrates a CPU-vs-GPU speed ratio in the reference
        # (partition.py:157-190); identical B200 parts always balance at 0.5.
        if cfg.ratio == "auto":
            warnings.warn("ratio='auto' calibrates a CPU/GPU speed ratio in the reference; every part is an "
                          "identical B200 here, so the split is 0.5", stacklevel=3)
        ratio = 0.5 if cfg.ratio == "auto" else float(cfg.ratio)
        return greedy_bipartition(g, ratio, seed=cfg.seed)
    return block_partition(g, cfg.num_partitions)


def default_groups(g: Graph, n_sources: int) -> int:
    """Source groups per batch: enough lanes to fill the GPU on small graphs,
    few enough that one group's sigma slab stays L2-friendly on large ones."""
    want = max(1, (n_sources + 31) // 32)
    # batch state out of 180 GB HBM: ~64 GB on shallow (high-degree) graphs at 600 B per vertex and
    # group (sigma + coef rows, masks); low-degree (deep) graphs sweep on frontier queues over
    # level-ordered values on top of the rows -- ~1,400 B per vertex and group, ~96 GB
    shallow = g.num_arcs >= 8 * g.num_vertices
    budget = max(1, int(64e9 // max(1, g.num_vertices * 600)) if shallow
                 else int(96e9 // max(1, g.num_vertices * 1400)))
    cap = min(budget, 32 if g.num_arcs >= 8_000_000 else 128)
    batches = (want + cap - 1) // cap
    return max(1, (want + batches - 1) // batches)               # batches of equal size


def open_engine(g: Graph, cfg: RunConfig, n_sources: int) -> _capi.Engine:
    device = cfg.device
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    eng = _capi.Engine(g, device)
    eng.set_option("groups", cfg.groups or default_groups(g, n_sources))
    if cfg.item_arcs:
        eng.set_option("item_arcs", cfg.item_arcs)
    eng.set_option("reports", 1 if cfg.per_source_reports else 0)
    return eng


def prepare(g: Graph, cfg: RunConfig):
    """Partition and borders (engine.py:87-102); border tables live on the device."""
    p = make_partition(g, cfg)
    bs = identify_borders(g, p)
    return p, bs


def border_table_bytes(bs: BorderSet) -> float:
    """Device bytes of the border tables: per part b_p x b_p entries of int32 distance + fp64
    path count (the b^2 term of the reference's memory model, border_matrix.py:70-82)."""
    return float(sum(12.0 * b * b for b in bs.counts()))


GENERAL_WEIGHT_LIMIT = 4096   # largest arc weight of the level-per-distance kernels (bc_set_weights)


def choose_mode(mode: str, bs: BorderSet, budget_bytes: float) -> str:
    """``hybir`` needs the border tables; when they do not fit the budget the run falls back to
    the reference's other partitioned mode, which is pinned to give the same BC
    (test_acceptance.py:288-297) and needs no tables (SURVEY.md hard part 2)."""
    if mode == "hybir" and border_table_bytes(bs) > budget_bytes:
        warnings.warn("border tables need %.1f GB (borders per part: %s), above the %.1f GB budget: "
                      "running mode 'bsp-baseline' instead of 'hybir'"
                      % (border_table_bytes(bs) / 1e9, list(bs.counts()), budget_bytes / 1e9), stacklevel=3)
        return "bsp-baseline"
    return mode


def _table_cache_path(g: Graph, p: Partition, cache_dir: str) -> str:
    h = hashlib.sha256()
    h.update(g.content_hash().encode())
    h.update(np.ascontiguousarray(p.assignment, dtype=np.int32).tobytes())
    return os.path.join(cache_dir, "border_tables_%s.npz" % h.hexdigest()[:32])


def load_border_tables(eng, g: Graph, p: Partition, bs: BorderSet, cache_dir: str) -> bool:
    """Install cached border tables (keyed by graph + partition); False when there is no match."""
    path = _table_cache_path(g, p, cache_dir)
    try:
        data = np.load(path)
    except (OSError, ValueError):
        return False
    counts = bs.counts()
    if int(data["version"]) != 1 or list(data["counts"]) != list(counts):
        return False
    for part, b in enumerate(counts):
        eng.set_border_tables(part, data["bm%d" % part], data["sm%d" % part])
    return True


def save_border_tables(eng, g: Graph, p: Partition, bs: BorderSet, cache_dir: str) -> str:
    os.makedirs(cache_dir, exist_ok=True)
    path = _table_cache_path(g, p, cache_dir)
    arrays = {"version": np.int64(1), "counts": np.asarray(bs.counts(), dtype=np.int64)}
    for part, b in enumerate(bs.counts()):
        _, bm, sm = eng.border_tables(part, b)
        arrays["bm%d" % part], arrays["sm%d" % part] = bm, sm
    tmp = path + ".tmp.npz"
    np.savez(tmp, **arrays)
    os.replace(tmp, path)
    return path


def _per_source(sources, reports, mode):
    out = []
    for s, r in zip(sources, reports):
        it, ce, ml0, ml1, se, cb, l0, l1 = (int(x) for x in r)
        if mode == "bsp-baseline":
            fwd = {"source": int(s), "supersteps": it, "comm_events": ce, "max_level": [ml0, ml1]}
        else:
            fwd = {"source": int(s), "iterations": it, "comm_events": ce, "max_level": [ml0, ml1]}
        bwd = {"sync_events": se, "comm_bytes": cb, "levels": [l0, l1]}
        out.append({"source": int(s), "forward": fwd, "backward": bwd})
    return out


def run_bc(g: Graph, cfg: RunConfig | None = None, _pipeline: bool = False) -> RunResult:
    cfg = cfg or RunConfig()
    if g.num_vertices == 0:
        raise InputError("empty graph")
    if not g.unit_weight and cfg.num_gpus > 1 and cfg.gpu_mode == "graph-partitioned":
        # weighted graphs (positive integer weights) run level = distance sweeps in every
        # single-GPU mode; the multi-GPU border exchange is unit-weight
        raise InputError("weighted graph: use gpu_mode='source-sharded'")
    if cfg.num_gpus > 1:
        from .multigpu import run_bc_multi
        return run_bc_multi(g, cfg)
    t0 = time.perf_counter()
    sources = select_sources(g, cfg)
    p, bs = prepare(g, cfg)
    mode = choose_mode(cfg.mode, bs, cfg.table_budget_bytes) if p.num_parts > 1 else "direct"
    if mode != "direct" and not g.unit_weight and int(g.arc_weight.max()) > GENERAL_WEIGHT_LIMIT:
        # the partitioned modes take one level per distance value; beyond that the engine has the
        # label-correcting sweeps of csrc/bc_sssp.cuh, which are unpartitioned (same BC)
        warnings.warn("arc weights above %d: running mode 'direct' instead of '%s'"
                      % (GENERAL_WEIGHT_LIMIT, mode), stacklevel=2)
        mode = "direct"
    with open_engine(g, cfg, len(sources)) as eng:
        if p.num_parts > 1 and mode != "direct":
            eng.set_partition(p.num_parts, p.assignment)
        cached = False
        if mode == "hybir" and cfg.table_cache_dir:
            cached = load_border_tables(eng, g, p, bs, cfg.table_cache_dir)
        if _pipeline:
            eng.set_option("lookahead", 1)
        bc, stats = eng.run(sources, _MODE_CODE[mode])
        stats["mode"] = mode
        stats["border_tables_from_cache"] = cached
        if mode == "hybir" and cfg.table_cache_dir and not cached:
            save_border_tables(eng, g, p, bs, cfg.table_cache_dir)
        per_source = []
        if cfg.per_source_reports and p.num_parts > 1 and mode != "direct":
            per_source = _per_source(sources, eng.reports(len(sources)), mode)
        elif cfg.per_source_reports:
            per_source = [{"source": int(s), "forward": {"source": int(s)}, "backward": {}} for s in sources]
    elapsed = time.perf_counter() - t0
    mteps = (g.num_edges * len(sources) / elapsed / 1e6) if elapsed > 0 else 0.0
    ledger = CommTotals(stats.get("comm_events", 0), stats.get("sync_events", 0),
                        stats.get("comm_bytes", 0))
    return RunResult(bc, per_source, ledger, mteps, elapsed, p, bs, cfg,
                     int(stats.get("lookahead_batches", 0)), stats)


def pipeline_sources(g: Graph, cfg: RunConfig) -> RunResult:
    """Look-ahead variant (engine.py:135-143,156-161): Step 1 of the NEXT source batch runs on a
    second CUDA stream while the border refinement / path-count composition of the current
    batch is in flight (it only needs the BFS state, which the border phase does not touch);
    ``pipeline_overlaps`` counts the batches whose Step 1 was issued ahead.  Same result as
    ``run_bc`` (test_engine.py:57-64): bit for bit on the row layout, up to the rounding order of
    the atomically accumulated BC vector on deep graphs (level-ordered sweeps).  On one GPU the
    overlap buys no device time -- Step 1 and the border phase compete for the same memory system
    (road-like 2048^2 in 8 strips, 4 batches: 1,309 vs 1,298 ms) -- it is there for interface parity
    and for ranks whose border phase waits on collectives."""
    if cfg.mode != "hybir":
        raise InputError("pipelining applies to hybir mode only")
    return run_bc(g, cfg, _pipeline=True)


def build_report(g: Graph, result: RunResult, top_k: int = 10) -> dict:
    """JSON-ready report with the reference's field order (engine.py:164-189)."""
    bc = result.bc
    order = np.argsort(-bc, kind="stable")[:top_k]
    return {
        "schema_version": 1,
        "graph_stats": graph_stats(g),
        "partition_stats": {
            "sizes": list(result.partition.sizes),
            "ratio": result.partition.ratio,
            "borders": list(result.borders.counts()),
            "cut_arcs": len(result.borders.cut_src),
        },
        "mode": result.config.mode,
        "seed": result.config.seed,
        "per_source": result.per_source,
        "comm_totals": result.ledger.totals(),
        "bc_top_k": [{"vertex": int(v), "bc": float(bc[v])} for v in order],
        "mteps": result.mteps,
        "pipeline_overlaps": result.pipeline_overlaps,
        "max_threads": result.config.max_threads,
    }

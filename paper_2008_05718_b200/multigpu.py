"""One-process-per-GPU execution over ``torch.distributed`` (NCCL / NVLink).

Source-sharded mode: the CSR is replicated on every
GPU, the source list is dealt round-robin to the ranks, every rank
accumulates a local BC vector on its device and ONE ``all_reduce(SUM)`` of
that fp64 vector ends the job.  Sources are independent (the reference's
source loop is a plain sum, engine.py:132-149), so there is no other
collective on the data path; BC differs from the single-GPU result by
summation order only.

torch is used for plumbing only (process group, the device vector that NCCL
reduces, the CUDA stream handed to the C ABI).
"""

from __future__ import annotations

import os
import time

import numpy as np

from .errors import EngineError, InputError

__all__ = ["shard_sources", "init_process_group", "run_bc_multi", "sharded_bc"]


def shard_sources(sources, rank: int, world: int) -> list:
    """Round-robin deal: rank r takes sources[r], sources[r + world], ..."""
    if not 0 <= rank < world:
        raise InputError("rank %d outside world of %d" % (rank, world))
    return list(sources[rank::world])


def init_process_group(backend: str | None = None):
    """Join the job torchrun started (RANK / WORLD_SIZE / MASTER_* in the env)."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    if "RANK" not in os.environ or "WORLD_SIZE" not in os.environ:
        raise EngineError("multi-GPU runs are launched one process per GPU "
                          "(torchrun / torch.distributed.run sets RANK and WORLD_SIZE)")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29500")
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group(backend=backend)
    return dist.get_rank(), dist.get_world_size()


def sharded_bc(n: int, sources, compute_local, device="cuda"):
    """Deal ``sources`` over the ranks, run ``compute_local(shard, bc_tensor)``
    (which must ADD its shard's contribution into ``bc_tensor``, an fp64
    vector on ``device``), then all-reduce.  Returns the reduced tensor."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    bc = torch.zeros(n, dtype=torch.float64, device=device)
    compute_local(shard_sources(list(sources), rank, world), bc)
    dist.all_reduce(bc, op=dist.ReduceOp.SUM)
    return bc


def run_bc_multi(g, cfg):
    """``run_bc`` on ``cfg.num_gpus`` ranks; every rank returns the full BC vector."""
    import torch
    import torch.distributed as dist

    from . import _capi
    from .engine import (GENERAL_WEIGHT_LIMIT, CommTotals, RunResult, _MODE_CODE, open_engine, prepare,
                         select_sources)

    rank, world = init_process_group()
    if world != cfg.num_gpus:
        raise InputError("cfg.num_gpus=%d but the process group has %d ranks" % (cfg.num_gpus, world))
    if cfg.gpu_mode == "graph-partitioned":
        from .partitioned import run_bc_partitioned
        return run_bc_partitioned(g, cfg)
    if not torch.cuda.is_available():
        raise EngineError("no CUDA device: the BC engine has no CPU fallback")

    t0 = time.perf_counter()
    sources = select_sources(g, cfg)
    p, bs = prepare(g, cfg)
    mode = cfg.mode if p.num_parts > 1 else "direct"
    if mode != "direct" and not g.unit_weight and int(g.arc_weight.max()) > GENERAL_WEIGHT_LIMIT:
        mode = "direct"     # general-weight sweeps are unpartitioned (run_bc warns about the same step)
    # the BC vector NCCL reduces must live on the device the engine runs on (open_engine's rule)
    ordinal = cfg.device if cfg.device is not None else int(os.environ.get("LOCAL_RANK", "0"))
    device = torch.device("cuda", ordinal)
    torch.cuda.set_device(device)
    stats = {}
    with open_engine(g, cfg, (len(sources) + world - 1) // world) as eng:
        if p.num_parts > 1 and mode != "direct":
            eng.set_partition(p.num_parts, p.assignment)

        def compute_local(shard, bc_tensor):
            stream = torch.cuda.current_stream(device).cuda_stream
            stats.update(eng.run_device(shard, bc_tensor.data_ptr(), stream, _MODE_CODE[mode]))

        bc = sharded_bc(g.num_vertices, sources, compute_local, device)
        bc_host = bc.cpu().numpy()
    elapsed = time.perf_counter() - t0
    mteps = g.num_edges * len(sources) / elapsed / 1e6 if elapsed > 0 else 0.0
    ledger = CommTotals(stats.get("comm_events", 0), stats.get("sync_events", 0),
                        stats.get("comm_bytes", 0))
    return RunResult(bc_host, [], ledger, mteps, elapsed, p, bs, cfg, 0, stats)

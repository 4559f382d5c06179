"""Graph-partitioned multi-GPU mode: one rank = one part = one GPU.

The paper's fine-grained mode with the CPU part replaced by further GPU parts
(SURVEY.md section 8e).  Every rank holds the CSR rows of its own vertices;
sources advance 32 x groups at a time, level-synchronously (the reference's
bsp schedule, bsp.py:22-142), and the only data that crosses NVLink is what
the reference's ledger counts as cross-worker transfers: after forward level L
the level masks and path counts of the *border* vertices discovered at L,
after backward level L the (1 + delta) / sigma values of the border vertices
sitting at L.  Collectives per level: one all-gather of the border masks, one
all-gather of the lane-compacted values, one tiny all-gather of the
live-lane words.  BC ends with one all-reduce (each vertex has one owner, the
other ranks contribute zeros).

torch.distributed is plumbing: NCCL on CUDA tensors in production; with the
gloo backend (tests: two ranks sharing one GPU) the same buffers are staged
through host memory.
"""

from __future__ import annotations

import os
import time

import numpy as np

from .errors import EngineError, InputError
from .graph import Graph
from .partition import Partition, block_partition, identify_borders

__all__ = ["local_rows", "run_bc_partitioned", "PartitionedRunner"]


def local_rows(g: Graph, assignment, rank: int) -> Graph:
    """The rank's CSR: adjacency of its own vertices, empty rows elsewhere
    (global vertex ids are kept, so state arrays line up across ranks)."""
    own = np.asarray(assignment) == rank
    deg = np.diff(g.offsets) * own
    offsets = np.zeros(g.num_vertices + 1, dtype=np.int64)
    np.cumsum(deg, out=offsets[1:])
    keep = np.repeat(own, np.diff(g.offsets))
    col = g.col_idx[keep]
    return Graph(g.num_vertices, len(col) // 2, offsets, col)


class _Transport:
    """all-gather of equally sized device buffers over NCCL, or staged through
    the host when the process group is gloo."""

    def __init__(self, device):
        import torch.distributed as dist
        self.dist = dist
        self.device = device
        self.world = dist.get_world_size()
        self.on_device = dist.get_backend() == "nccl"

    def all_gather(self, t):
        import torch
        if self.on_device:
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t.contiguous())
            return out
        host = t.cpu()
        parts = [torch.empty_like(host) for _ in range(self.world)]
        self.dist.all_gather(parts, host)
        return torch.stack(parts).to(self.device)

    def all_reduce_sum(self, t):
        if self.on_device:
            self.dist.all_reduce(t)
            return t
        host = t.cpu()
        self.dist.all_reduce(host)
        t.copy_(host)
        return t


class PartitionedRunner:
    def __init__(self, g: Graph, part: Partition, device, groups: int = 4):
        import torch
        import torch.distributed as dist
        from . import _capi

        self.torch = torch
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if part.num_parts != self.world:
            raise InputError("graph-partitioned mode needs one part per rank (%d parts, %d ranks)"
                             % (part.num_parts, self.world))
        self.g, self.part, self.device, self.groups = g, part, device, groups
        self.n = g.num_vertices
        bs = identify_borders(g, part)
        self.border_counts = [len(b) for b in bs.border_arrays]
        self.border_off = np.concatenate(([0], np.cumsum(self.border_counts))).astype(np.int64)
        border_v = (np.concatenate(bs.border_arrays) if sum(self.border_counts)
                    else np.zeros(0, dtype=np.int64)).astype(np.int32)
        self.eng = _capi.Engine(local_rows(g, part.assignment, self.rank), device.index or 0)
        self.eng.set_option("groups", groups)
        self.eng.dist_setup(self.rank, self.world, part.assignment, self.border_off, border_v)
        self.tr = _Transport(device)
        self.max_nb = max(self.border_counts + [1])
        self.stream = 0     # default stream: exports / imports and collectives stay ordered
        self.exchanged_bytes = 0
        self.levels = 0

    def close(self):
        self.eng.close()

    def _exchange(self, level, what, ng):
        torch = self.torch
        entries = self.max_nb * ng
        masks = torch.zeros(entries, dtype=torch.int32, device=self.device)
        values = torch.empty(max(entries * 32, 1), dtype=torch.float64, device=self.device)
        count = self.eng.dist_export(level, what, masks.data_ptr(), values.data_ptr(), values.numel())
        counts = self.tr.all_gather(torch.tensor([count], dtype=torch.int64, device=self.device)).view(-1)
        widest = int(counts.max().item())
        all_masks = self.tr.all_gather(masks)
        all_values = self.tr.all_gather(values[:max(widest, 1)])
        self.exchanged_bytes += masks.numel() * 4 + count * 8
        for peer in range(self.world):
            if peer == self.rank or self.border_counts[peer] == 0:
                continue
            # a peer's block is laid out [its nb][ng]; our padding sits at the tail
            self.eng.dist_import(level, what, peer, all_masks[peer].data_ptr(),
                                 all_values[peer].data_ptr())
        self.torch.cuda.synchronize(self.device)   # buffers are freed on return

    def run_batch(self, sources):
        torch = self.torch
        ng = (len(sources) + 31) // 32
        self.eng.dist_begin(sources)
        depth = 1
        level = 1
        while True:
            self.eng.dist_forward_level(level)
            if self.world > 1:
                self._exchange(level, 1, ng)
            live = torch.from_numpy(self.eng.dist_get_live(level, ng).astype(np.int64)).to(self.device)
            if self.world > 1:
                live = self.tr.all_gather(live)
                merged = live[0]
                for r in range(1, self.world):
                    merged = merged | live[r]
                live = merged
            live_host = live.cpu().numpy().astype(np.uint32)
            self.eng.dist_set_live(level, live_host)
            if not live_host.any():
                depth = level
                break
            level += 1
        for lv in range(depth - 1, 0, -1):
            self.eng.dist_backward_level(lv, lv == depth - 1)
            if self.world > 1 and lv > 1:
                self._exchange(lv, 2, ng)
        self.levels = max(self.levels, depth)
        return depth

    def run(self, sources):
        torch = self.torch
        bc = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        per = 32 * self.groups
        for lo in range(0, len(sources), per):
            self.run_batch(list(sources[lo:lo + per]))
        self.eng.dist_finish(bc.data_ptr())
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            self.tr.all_reduce_sum(bc)
        return bc


def run_bc_partitioned(g: Graph, cfg):
    """``run_bc`` with ``gpu_mode='graph-partitioned'``: every rank returns the full BC vector."""
    import torch
    import torch.distributed as dist

    from .engine import CommTotals, RunResult, select_sources
    from .multigpu import init_process_group

    rank, world = init_process_group()
    if not torch.cuda.is_available():
        raise EngineError("no CUDA device: the BC engine has no CPU fallback")
    t0 = time.perf_counter()
    device = torch.device("cuda", cfg.device if cfg.device is not None
                          else int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(device)
    part = cfg.partition if cfg.partition is not None else block_partition(g, world)
    sources = select_sources(g, cfg)
    runner = PartitionedRunner(g, part, device, cfg.groups or 4)
    try:
        bc = runner.run(sources).cpu().numpy()
    finally:
        runner.close()
    elapsed = time.perf_counter() - t0
    bs = identify_borders(g, part)
    stats = {"levels": runner.levels, "exchanged_bytes": runner.exchanged_bytes, "world": world}
    mteps = g.num_edges * len(sources) / elapsed / 1e6 if elapsed > 0 else 0.0
    return RunResult(bc, [], CommTotals(0, 0, runner.exchanged_bytes), mteps, elapsed, part, bs, cfg,
                     0, stats)

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
        return self.all_reduce(t, "sum")

    def all_reduce(self, t, op: str):
        red = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN,
               "max": self.dist.ReduceOp.MAX}[op]
        if self.on_device:
            self.dist.all_reduce(t, op=red)
            return t
        host = t.cpu()
        self.dist.all_reduce(host, op=red)
        t.copy_(host)
        return t

    def broadcast(self, t, src: int):
        if self.on_device:
            self.dist.broadcast(t, src=src)
            return t
        host = t.cpu()
        self.dist.broadcast(host, src=src)
        t.copy_(host)
        return t


def incoming_cut_arcs(bs, border_arrays):
    """(cin_off, cin_src): for every border, in the rank-major border order, the border
    indices on the other side of its cut arcs (the graph is symmetric, so the incoming arcs
    of a border are its own cut arcs reversed)."""
    total = int(sum(len(b) for b in border_arrays))
    cin_off = np.zeros(total + 1, dtype=np.int64)
    if total == 0 or len(bs.cut_src) == 0:
        return cin_off, np.zeros(0, dtype=np.int32)
    all_borders = np.concatenate(border_arrays).astype(np.int64)
    index_of = np.full(int(max(all_borders.max(), np.max(bs.cut_dst))) + 1, -1, dtype=np.int64)
    index_of[all_borders] = np.arange(total)
    at = index_of[np.asarray(bs.cut_src, dtype=np.int64)]
    other = index_of[np.asarray(bs.cut_dst, dtype=np.int64)]
    order = np.argsort(at, kind="stable")
    np.cumsum(np.bincount(at, minlength=total), out=cin_off[1:])
    return cin_off, other[order].astype(np.int32)


class PartitionedRunner:
    """``forward='bsp'``: level-synchronous forward phase, one border exchange per level
    (bsp.py:22-103).  ``forward='hybir'``: the paper's border-matrix forward phase
    (forward.py:188-256) -- Step 1 inside the source's part, ONE exchange of the border
    seeds, refinement + path-count composition on the border tables (replicated on every
    rank), Step 6 inside every part; the forward phase of a batch then costs two all-reduces
    whatever the diameter.  The backward phase is level-synchronous in both."""

    def __init__(self, g: Graph, part: Partition, device, groups: int = 4, forward: str = "bsp"):
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
        if forward not in ("bsp", "hybir"):
            raise InputError("forward must be 'bsp' or 'hybir'")
        self.forward = forward
        self.iterations = 0
        self.forward_exchanges = 0
        self.backward_exchanges = 0
        if forward == "hybir":
            if not g.unit_weight:
                raise InputError("the multi-GPU border exchange is unit-weight")
            cin_off, cin_src = incoming_cut_arcs(bs, bs.border_arrays)
            self.eng.dist_hybir_setup(cin_off, cin_src)
            # every rank publishes the border table of its own part once
            for p in range(self.world):
                b = self.border_counts[p]
                if b == 0:
                    continue
                bm = torch.empty(b * b, dtype=torch.int32, device=device)
                sm = torch.empty(b * b, dtype=torch.float64, device=device)
                if p == self.rank:
                    self.eng.dist_hybir_get_table(p, bm.data_ptr(), sm.data_ptr())
                if self.world > 1:
                    self.tr.broadcast(bm, p)
                    self.tr.broadcast(sm, p)
                if p != self.rank:
                    self.eng.dist_hybir_set_table(p, bm.data_ptr(), sm.data_ptr())
                torch.cuda.synchronize(device)
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

    def _forward_hybir(self, sources):
        torch = self.torch
        cnt = self.eng.dist_hybir_seed_count()
        sd = torch.empty(max(cnt, 1), dtype=torch.int32, device=self.device)
        ss = torch.empty(max(cnt, 1), dtype=torch.float64, device=self.device)
        self.eng.dist_hybir_seeds(sources, sd.data_ptr(), ss.data_ptr())
        if self.world > 1:
            # only the rank that owns a lane's source holds finite seeds for that lane
            self.tr.all_reduce(sd, "min")
            self.tr.all_reduce(ss, "max")
            self.forward_exchanges += 2
            self.exchanged_bytes += cnt * 12
        depth, iters = self.eng.dist_hybir_forward(sd.data_ptr(), ss.data_ptr())
        self.iterations += iters
        d = torch.tensor([depth], dtype=torch.int64, device=self.device)
        if self.world > 1:
            self.tr.all_reduce(d, "max")
        depth = int(d.item())
        self.eng.dist_hybir_set_depth(depth)
        torch.cuda.synchronize(self.device)
        return depth

    def run_batch(self, sources):
        torch = self.torch
        ng = (len(sources) + 31) // 32
        if self.forward == "hybir":
            depth = self._forward_hybir(sources)
            for lv in range(depth - 1, 0, -1):
                self.eng.dist_backward_level(lv, lv == depth - 1)
                if self.world > 1 and lv > 1:
                    self._exchange(lv, 2, ng)
                    self.backward_exchanges += 1
            self.levels = max(self.levels, depth)
            return depth
        self.eng.dist_begin(sources)
        depth = 1
        level = 1
        while True:
            self.eng.dist_forward_level(level)
            if self.world > 1:
                self._exchange(level, 1, ng)
                self.forward_exchanges += 1
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
                self.backward_exchanges += 1
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
    # RunConfig.mode picks the forward phase as in the reference: 'hybir' = border matrices
    # (weighted graphs and 'direct' fall back to the level-synchronous exchange)
    forward = "hybir" if (cfg.mode == "hybir" and g.unit_weight) else "bsp"
    runner = PartitionedRunner(g, part, device, cfg.groups or 4, forward)
    try:
        bc = runner.run(sources).cpu().numpy()
    finally:
        runner.close()
    elapsed = time.perf_counter() - t0
    bs = identify_borders(g, part)
    stats = {"levels": runner.levels, "exchanged_bytes": runner.exchanged_bytes, "world": world,
             "forward": runner.forward, "forward_exchanges": runner.forward_exchanges,
             "backward_exchanges": runner.backward_exchanges, "iterations": runner.iterations}
    mteps = g.num_edges * len(sources) / elapsed / 1e6 if elapsed > 0 else 0.0
    return RunResult(bc, [], CommTotals(0, 0, runner.exchanged_bytes), mteps, elapsed, part, bs, cfg,
                     0, stats)

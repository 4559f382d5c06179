"""Graph-partitioned multi-GPU mode: one rank = one part = one GPU.

The paper's fine-grained mode with the CPU part replaced by further GPU parts
(SURVEY.md section 8e).  Every rank holds the CSR rows of its own vertices and
state arrays over its own vertices plus a *halo* -- the other parts' border
vertices its cut arcs reach (``local_graph``); nothing on a rank is sized by
the whole graph except the final BC vector.  Sources advance 32 x groups at a
time.

Forward phase, chosen by ``RunConfig.mode`` as in the reference:
  ``hybir``         the paper's border-matrix forward phase (forward.py:188-256):
                    Step 1 inside the source's part, ONE exchange of the border
                    seeds (two all-reduces per batch, whatever the diameter),
                    refinement + path-count composition on the border tables,
                    Step 6 inside every part
  ``bsp-baseline``  level-synchronous (bsp.py:22-103): after level L the level
                    masks and path counts of the border vertices found at L
Backward phase (backward.py:46-56,121-139): a rank only has to publish
``(1 + delta) / sigma`` of a border vertex at level L if a vertex of another
part at level L - 1 pulls it.  Those (border, lanes) values are listed level
by level ONCE per batch from the forward result (``bc_dist_plan_backward``,
one host round trip), the per-level counts are all-gathered once, and the
backward sweep then runs without any host synchronisation: at the levels some
rank has values to publish, one packed all-gather of exactly those values on
the stream the kernels run on; at all other levels nothing crosses.  BC ends
with one all-reduce (each vertex has one owner, the other ranks add zeros).

torch.distributed is plumbing: NCCL on CUDA tensors in production; with the
gloo backend (tests: ranks sharing one GPU) the same buffers are staged
through host memory.
"""

from __future__ import annotations

import os
import time

import numpy as np

from .errors import EngineError, InputError
from .graph import Graph
from .partition import Partition, block_partition, identify_borders

__all__ = ["local_rows", "local_graph", "LocalGraph", "run_bc_partitioned", "PartitionedRunner"]


def local_rows(g: Graph, assignment, rank: int) -> Graph:
    """The rank's rows in GLOBAL numbering: adjacency of its own vertices, empty rows elsewhere
    (kept for inspection; the runner uses ``local_graph``)."""
    own = np.asarray(assignment) == rank
    deg = np.diff(g.offsets) * own
    offsets = np.zeros(g.num_vertices + 1, dtype=np.int64)
    np.cumsum(deg, out=offsets[1:])
    keep = np.repeat(own, np.diff(g.offsets))
    col = g.col_idx[keep]
    return Graph(g.num_vertices, len(col) // 2, offsets, col)


class LocalGraph:
    """A rank's view of the partitioned graph, numbered locally:

    ``[0, n_own)``                 its own vertices, ascending global id (rows = their adjacency)
    ``[n_own, n_own + n_halo)``    halo: other parts' border vertices next to them (empty rows)
    then one catch-all vertex per other part for the borders this rank has no arc to (their
    level marks are never read here).

    ``border_v``: every rank's borders in local ids (rank-major, ascending global id per rank);
    ``cut_off / cut_dst``: cut arcs of the rank's own borders (far ends are halo vertices).
    """

    def __init__(self, g: Graph, part: Partition, bs, rank: int):
        a = np.asarray(part.assignment).astype(np.int64)
        n, k = g.num_vertices, part.num_parts
        self.rank, self.world = rank, k
        self.owned = np.flatnonzero(a == rank)
        n_own = len(self.owned)
        deg = np.diff(g.offsets)
        # adjacency of the owned vertices
        keep = np.repeat(a == rank, deg)
        col = g.col_idx[keep].astype(np.int64)
        off = np.zeros(n_own + 1, dtype=np.int64)
        np.cumsum(deg[self.owned], out=off[1:])
        foreign = a[col] != rank
        halo = np.unique(col[foreign])                       # ascending global id
        # rank-major order, as the border lists are
        halo = halo[np.argsort(a[halo], kind="stable")]
        n_halo = len(halo)
        others = [q for q in range(k) if q != rank]
        self.n_own, self.n_halo = n_own, n_halo
        self.n_local = n_own + n_halo + len(others)
        self.halo = halo
        local_of = np.full(n, -1, dtype=np.int64)
        local_of[self.owned] = np.arange(n_own)
        local_of[halo] = n_own + np.arange(n_halo)
        self.local_of = local_of
        catch_all = {q: n_own + n_halo + i for i, q in enumerate(others)}
        self.catch_all = catch_all
        offsets = np.concatenate([off, np.full(self.n_local - n_own, off[-1], dtype=np.int64)])
        col_local = local_of[col]
        self.graph = Graph(self.n_local, len(col_local) // 2, offsets, col_local.astype(np.int32))
        assign = np.empty(self.n_local, dtype=np.int32)
        assign[:n_own] = rank
        assign[n_own:n_own + n_halo] = a[halo]
        for q, v in catch_all.items():
            assign[v] = q
        self.assignment = assign
        # border lists
        border_v = []
        for q, b in enumerate(bs.border_arrays):
            lv = local_of[np.asarray(b, dtype=np.int64)]
            if q != rank:
                lv = np.where(lv < 0, catch_all.get(q, 0), lv)
            border_v.append(lv)
        self.border_counts = [len(b) for b in bs.border_arrays]
        self.border_off = np.concatenate(([0], np.cumsum(self.border_counts))).astype(np.int64)
        self.border_v = (np.concatenate(border_v) if sum(self.border_counts) else
                         np.zeros(0, dtype=np.int64)).astype(np.int32)
        # cut arcs of the own borders, in border order
        mine = np.asarray(bs.border_arrays[rank], dtype=np.int64)
        src = np.asarray(bs.cut_src, dtype=np.int64)
        sel = a[src] == rank if len(src) else np.zeros(0, dtype=bool)
        cs, cd = src[sel], np.asarray(bs.cut_dst, dtype=np.int64)[sel]
        pos = np.searchsorted(mine, cs)                      # bs.cut_* is sorted by (src, dst)
        self.cut_off = np.zeros(len(mine) + 1, dtype=np.int64)
        if len(cs):
            np.cumsum(np.bincount(pos, minlength=len(mine)), out=self.cut_off[1:])
        self.cut_dst = local_of[cd].astype(np.int32)


def local_graph(g: Graph, part: Partition, rank: int, bs=None) -> LocalGraph:
    return LocalGraph(g, part, bs if bs is not None else identify_borders(g, part), rank)


class _Transport:
    """Collectives over equally sized device buffers: NCCL in place, or staged through the host
    when the process group is gloo."""

    def __init__(self, device):
        import torch.distributed as dist
        self.dist = dist
        self.device = device
        self.world = dist.get_world_size()
        self.on_device = dist.get_backend() == "nccl"

    def all_gather_into(self, out, t):
        """out[world * len(t)] <- every rank's t (out / t are preallocated views)."""
        import torch
        if self.on_device:
            self.dist.all_gather_into_tensor(out, t)
            return out
        host = t.cpu()
        parts = [torch.empty_like(host) for _ in range(self.world)]
        self.dist.all_gather(parts, host)
        out.copy_(torch.cat(parts).to(self.device))
        return out

    def all_gather(self, t):
        import torch
        out = torch.empty((self.world * t.numel(),), dtype=t.dtype, device=t.device)
        return self.all_gather_into(out, t.contiguous().view(-1)).view((self.world,) + tuple(t.shape))

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
    """One rank of a graph-partitioned run (see the module docstring)."""

    def __init__(self, g: Graph, part: Partition, device, groups: int = 4, forward: str = "bsp",
                 shard_tables: bool = True):
        import torch
        import torch.distributed as dist
        from . import _capi

        self.torch = torch
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if part.num_parts != self.world:
            raise InputError("graph-partitioned mode needs one part per rank (%d parts, %d ranks)"
                             % (part.num_parts, self.world))
        if forward not in ("bsp", "hybir"):
            raise InputError("forward must be 'bsp' or 'hybir'")
        if not g.unit_weight:
            # the level kernels of this mode and the border exchange are unit-weight
            raise InputError("weighted graph: use gpu_mode='source-sharded'")
        self.g, self.part, self.device, self.groups = g, part, device, groups
        self.n = g.num_vertices
        self.assignment = np.asarray(part.assignment).astype(np.int32)
        bs = identify_borders(g, part)
        self.lg = LocalGraph(g, part, bs, self.rank)
        self.local_n = self.lg.n_local
        self.border_counts = list(self.lg.border_counts)
        self.eng = _capi.Engine(self.lg.graph, device.index or 0)
        self.eng.set_option("groups", groups)
        self.eng.dist_setup(self.rank, self.world, self.lg.assignment, self.lg.border_off, self.lg.border_v)
        self.eng.dist_set_cut_arcs(self.lg.cut_off, self.lg.cut_dst)
        self.tr = _Transport(device)
        self.forward = forward
        self.shard_tables = bool(shard_tables) and forward == "hybir" and self.world > 1
        if forward == "hybir":
            cin_off, cin_src = incoming_cut_arcs(bs, bs.border_arrays)
            self.eng.dist_hybir_setup(cin_off, cin_src)
            if self.shard_tables:
                # one table per rank: refinement / composition of a part run on its owner, the
                # border state is all-reduced after every iteration (_border_phase_sharded)
                self.eng.dist_hybir_shard_tables()
            # (replicated tables) every rank publishes the border table of its own part once
            for p in range(self.world if not self.shard_tables else 0):
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
            cnt = self.eng.dist_hybir_seed_count()
            self.seed_d = torch.zeros(max(cnt, 1), dtype=torch.int32, device=device)
            self.seed_s = torch.zeros(max(cnt, 1), dtype=torch.float64, device=device)
            if self.shard_tables:
                self._xd = torch.zeros(max(cnt, 1), dtype=torch.int32, device=device)
                self._xs = torch.zeros(max(cnt, 1), dtype=torch.float64, device=device)
                self._xf = torch.zeros(32 * groups, dtype=torch.int32, device=device)
        self.max_nb = max(self.border_counts + [1])
        self.stream = 0     # default stream: kernels, packs / unpacks and collectives stay ordered
        # forward (bsp) exchange buffers, grown on demand and kept
        self._masks = torch.zeros(self.max_nb * groups, dtype=torch.int32, device=device)
        self._all_masks = torch.zeros(self.world * self.max_nb * groups, dtype=torch.int32, device=device)
        self._values = torch.zeros(max(self.max_nb * groups * 32, 1), dtype=torch.float64, device=device)
        self._all_values = torch.zeros(1, dtype=torch.float64, device=device)
        # backward messages: [cap_values fp64][3 x cap_entries int32] as one int64 buffer
        self._send = torch.zeros(1, dtype=torch.int64, device=device)
        self._recv = torch.zeros(1, dtype=torch.int64, device=device)
        self._counts = torch.zeros(1, dtype=torch.int64, device=device)
        self.levels = 0
        self.reset_counters()

    # -- bookkeeping ---------------------------------------------------------------------------
    def reset_counters(self):
        self.iterations = 0
        self.forward_exchanges = 0
        self.backward_exchanges = 0
        self.backward_levels = 0
        self.exchanged_bytes = 0
        self.eng.dist_stats()

    def counters(self) -> dict:
        st = self.eng.dist_stats()
        return {"forward_exchanges": self.forward_exchanges, "backward_exchanges": self.backward_exchanges,
                "backward_levels": self.backward_levels, "exchanged_bytes": self.exchanged_bytes,
                "iterations": self.iterations, "launches": st["launches"], "ms_level": st["ms_level"],
                "level_model_bytes": st["level_model_bytes"], "launches_level": st["launches_level"]}

    def close(self):
        self.eng.close()

    def _grown(self, t, count, dtype):
        if t.numel() < count:     # zero-filled: the padding of a message travels with it
            t = self.torch.zeros(int(count), dtype=dtype, device=self.device)
        return t

    # -- forward -------------------------------------------------------------------------------
    def _exchange_forward(self, level, ng):
        """bsp forward: masks + lane-compacted path counts of the borders found at `level`."""
        torch = self.torch
        entries = self.max_nb * ng
        masks = self._masks[:entries]
        masks.zero_()
        count = self.eng.dist_export(level, 1, masks.data_ptr(), self._values.data_ptr(), self._values.numel())
        counts = self.tr.all_gather(torch.tensor([count], dtype=torch.int64, device=self.device)).view(-1)
        widest = max(int(counts.max().item()), 1)
        all_masks = self._all_masks[:self.world * entries]
        self.tr.all_gather_into(all_masks, masks)
        self._all_values = self._grown(self._all_values, self.world * widest, torch.float64)
        all_values = self._all_values[:self.world * widest]
        self.tr.all_gather_into(all_values, self._values[:widest])
        self.exchanged_bytes += entries * 4 + count * 8
        for peer in range(self.world):
            if peer == self.rank or self.border_counts[peer] == 0:
                continue
            # a peer's block is laid out [its nb][ng]; our padding sits at the tail
            self.eng.dist_import(level, 1, peer, all_masks[peer * entries:].data_ptr(),
                                 all_values[peer * widest:].data_ptr())

    def _forward_bsp(self, local_src, ng):
        torch = self.torch
        self.eng.dist_begin(local_src)
        level = 1
        while True:
            self.eng.dist_forward_level(level)
            if self.world > 1:
                self._exchange_forward(level, ng)
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
                return level
            level += 1

    def _forward_hybir(self, local_src, src_part):
        torch = self.torch
        cnt = self.eng.dist_hybir_seed_count()
        sd, ss = self.seed_d, self.seed_s
        self.eng.dist_hybir_seeds(local_src, src_part, sd.data_ptr(), ss.data_ptr())
        if self.world > 1:
            # only the rank that owns a lane's source holds finite seeds for that lane
            self.tr.all_reduce(sd, "min")
            self.tr.all_reduce(ss, "max")
            self.forward_exchanges += 2
            self.exchanged_bytes += cnt * 12
        if self.shard_tables:
            depth = self._border_phase_sharded(sd, ss, cnt)
        else:
            depth, iters = self.eng.dist_hybir_forward(sd.data_ptr(), ss.data_ptr())
            self.iterations += iters
        d = torch.tensor([depth], dtype=torch.int64, device=self.device)
        if self.world > 1:
            self.tr.all_reduce(d, "max")
        depth = int(d.item())
        self.eng.dist_hybir_set_depth(depth)
        return depth

    def _border_phase_sharded(self, sd, ss, cnt):
        """Steps 2-5 + path-count composition with one border table per rank, then Step 6.  The
        "still active" flag is read back every 1, 1, 2, 3, 4, 4 ... iterations only (an iteration
        without active lanes changes nothing)."""
        eng, tr = self.eng, self.tr
        xd, xs, xf = self._xd, self._xs, self._xf
        eng.dist_hybir_border_step(0, seed_dist_ptr=sd.data_ptr(), seed_sigma_ptr=ss.data_ptr())
        total_borders = sum(self.border_counts)
        for compute, merge, values, op in ((1, 2, xd, "min"), (4, 5, xs, "max")):
            if compute == 4:
                eng.dist_hybir_border_step(3)
            it, poll = 0, 1
            while True:
                for j in range(poll):
                    eng.dist_hybir_border_step(compute, values.data_ptr(), xf.data_ptr())
                    tr.all_reduce(values, op)
                    tr.all_reduce(xf, "max")
                    self.forward_exchanges += 2
                    self.exchanged_bytes += cnt * (4 if compute == 1 else 8) + xf.numel() * 4
                    active = eng.dist_hybir_border_step(merge, values.data_ptr(), xf.data_ptr(),
                                                        want_flag=(j == poll - 1))
                    it += 1
                if compute == 1:
                    self.iterations += poll
                if not active:
                    break
                if it > 2 * total_borders + 16:
                    raise EngineError("border phase did not settle")
                poll = min(4, 1 + it // 2)
        return eng.dist_hybir_border_step(6, want_flag=True)

    # -- backward ------------------------------------------------------------------------------
    def _backward(self, depth, ng):
        """Level-reversed pull; border values cross only where the plan says another part pulls."""
        torch = self.torch
        plan = None
        if self.world > 1 and depth > 2:
            mine = torch.from_numpy(self.eng.dist_plan_backward(depth)).to(self.device)     # [depth, 2]
            plan_dev = self.tr.all_gather(mine).contiguous()                                # [world, depth, 2]
            plan = plan_dev.cpu().numpy()
            cap = plan.max(axis=0)                                                          # per level
            cap_e, cap_v = int(cap[:, 0].max()), int(cap[:, 1].max())
            words = cap_v + (3 * cap_e + 1) // 2                                            # int64 words per message
            self._send = self._grown(self._send, words, torch.int64)
            self._recv = self._grown(self._recv, self.world * words, torch.int64)
        for lv in range(depth - 1, 0, -1):
            self.eng.dist_backward_level(lv, lv == depth - 1)
            self.backward_levels += 1
            if plan is None or lv < 2 or plan[:, lv, 0].max() == 0:
                continue
            # one packed message per rank, sized by the largest sender of THIS level
            le, lvv = int(plan[:, lv, 0].max()), int(plan[:, lv, 1].max())
            words = lvv + (3 * le + 1) // 2
            send = self._send[:words]
            recv = self._recv[:self.world * words]
            self.eng.dist_pack(lv, send.data_ptr(), le, lvv)
            self.tr.all_gather_into(recv, send)
            # every peer's values land in the halo rows in one launch (counts read on the device)
            self.eng.dist_unpack_all(lv, recv.data_ptr(), words, le, lvv, plan_dev.data_ptr(), depth)
            self.backward_exchanges += 1
            self.exchanged_bytes += int(plan[self.rank, lv, 0]) * 12 + int(plan[self.rank, lv, 1]) * 8

    # -- driver --------------------------------------------------------------------------------
    def run_batch(self, sources):
        ng = (len(sources) + 31) // 32
        src = np.asarray(sources, dtype=np.int64)
        local_src = self.lg.local_of[src]
        if self.forward == "hybir":
            depth = self._forward_hybir(local_src, self.assignment[src])
        else:
            depth = self._forward_bsp(local_src, ng)
        self._backward(depth, ng)
        self.levels = max(self.levels, depth)
        return depth

    def run(self, sources):
        """BC over `sources`: the full vector, identical on every rank."""
        torch = self.torch
        local_bc = torch.zeros(self.local_n, dtype=torch.float64, device=self.device)
        per = 32 * self.groups
        for lo in range(0, len(sources), per):
            self.run_batch(list(sources[lo:lo + per]))
        self.eng.dist_finish(local_bc.data_ptr())
        bc = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        bc[torch.from_numpy(self.lg.owned).to(self.device)] = local_bc[:self.lg.n_own]
        if self.world > 1:
            self.tr.all_reduce_sum(bc)
        return bc


def run_bc_partitioned(g: Graph, cfg):
    """``run_bc`` with ``gpu_mode='graph-partitioned'``: every rank returns the full BC vector."""
    import torch

    from .engine import CommTotals, RunResult, border_table_bytes, choose_mode, select_sources
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
    bs = identify_borders(g, part)
    # RunConfig.mode picks the forward phase as in the reference: 'hybir' = border matrices (every
    # rank holds all parts' tables; above the budget the run falls back to the level-synchronous
    # exchange, as run_bc does); 'direct' has no partitioned meaning and takes the same fallback
    mode = choose_mode(cfg.mode, bs, cfg.table_budget_bytes) if cfg.mode == "hybir" else "bsp-baseline"
    forward = "hybir" if mode == "hybir" else "bsp"
    runner = PartitionedRunner(g, part, device, cfg.groups or 4, forward, cfg.shard_border_tables)
    try:
        bc = runner.run(sources).cpu().numpy()
        counters = runner.counters()
    finally:
        runner.close()
    elapsed = time.perf_counter() - t0
    stats = {"levels": runner.levels, "exchanged_bytes": runner.exchanged_bytes, "world": world,
             "forward": runner.forward, "forward_exchanges": runner.forward_exchanges,
             "backward_exchanges": runner.backward_exchanges, "backward_levels": runner.backward_levels,
             "iterations": runner.iterations, "state_vertices": runner.local_n,
             "owned_vertices": runner.lg.n_own, "halo_vertices": runner.lg.n_halo,
             "table_bytes": (0.0 if forward != "hybir" else
                             12.0 * runner.border_counts[rank] ** 2 if runner.shard_tables else border_table_bytes(bs)),
             "sharded_tables": runner.shard_tables,
             "launches": counters["launches"]}
    mteps = g.num_edges * len(sources) / elapsed / 1e6 if elapsed > 0 else 0.0
    return RunResult(bc, [], CommTotals(runner.forward_exchanges, runner.backward_exchanges,
                                        runner.exchanged_bytes), mteps, elapsed, part, bs, cfg, 0, stats)

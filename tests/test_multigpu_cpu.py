"""N>1 host logic on CPU: two gloo ranks deal the sources round-robin, each
computes its shard (the oracle stands in for the device engine here -- tests
may use it) and one all-reduce yields the full BC vector."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200.multigpu import shard_sources, sharded_bc


def test_shard_sources_is_a_partition():
    src = list(range(17))
    parts = [shard_sources(src, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == src
    assert parts[1] == [1, 5, 9, 13]
    assert shard_sources([3], 1, 2) == []


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = G.rmat(9, 6, 1)
    sources = list(range(0, g.num_vertices, 3))

    def compute_local(shard, bc_tensor):
        bc, _ = O.brandes_bc(g, shard, threads=1)
        bc_tensor += torch.from_numpy(bc)

    bc = sharded_bc(g.num_vertices, sources, compute_local, device="cpu")
    if rank == 0:
        full, _ = O.brandes_bc(g, sources, threads=1)
        np.save(out, np.stack([bc.numpy(), full]))
    dist.barrier()
    dist.destroy_process_group()


def test_source_sharded_allreduce_world2(tmp_path):
    out = str(tmp_path / "bc.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got, want = np.load(out)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    assert want.max() > 0


def _gp_worker(rank, world, port, out):
    """Host side of the graph-partitioned mode on CPU tensors: every rank numbers its part locally
    (own vertices + halo), the ranks exchange a per-level plan table and one packed message through
    the runner's transport, and scatter owned BC slices into the global vector."""
    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200.partitioned import LocalGraph, _Transport
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = G.grid(9, 8)
    part = P.strip_partition(9, 8, world)
    bs = P.identify_borders(g, part)
    lg = LocalGraph(g, part, bs, rank)
    tr = _Transport(torch.device("cpu"))
    # plan table [depth, 2] per rank -> [world, depth, 2]
    mine = torch.tensor([[rank + 1, 10 * (rank + 1)], [0, 0], [3, 7]], dtype=torch.int64)
    plan = tr.all_gather(mine)
    assert plan.shape == (world, 3, 2) and plan[:, 0, 0].tolist() == list(range(1, world + 1))
    # one packed message of equal size per rank
    words = int(plan[:, 2, 1].max()) + (3 * int(plan[:, 2, 0].max()) + 1) // 2
    send = torch.full((words,), rank, dtype=torch.int64)
    recv = torch.empty(world * words, dtype=torch.int64)
    tr.all_gather_into(recv, send)
    assert recv.view(world, words)[:, 0].tolist() == list(range(world))
    # owned slices of a local vector land in the global one; each vertex has one owner
    local = torch.arange(lg.n_local, dtype=torch.float64) + 1000.0 * rank
    bc = torch.zeros(g.num_vertices, dtype=torch.float64)
    bc[torch.from_numpy(lg.owned)] = local[:lg.n_own]
    tr.all_reduce_sum(bc)
    a = np.asarray(part.assignment)
    want = np.zeros(g.num_vertices)
    for r in range(world):
        own = np.flatnonzero(a == r)
        want[own] = np.arange(len(own)) + 1000.0 * r
    ok = bool(np.array_equal(bc.numpy(), want))
    # halo vertices of this rank are border vertices of their owners
    halo_ok = all(int(v) in set(np.asarray(bs.border_arrays[int(a[v])]).tolist()) for v in lg.halo)
    np.save("%s.%d.npy" % (out, rank), np.array([ok, halo_ok, lg.n_local, lg.n_own, lg.n_halo]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_graph_partitioned_host_logic_gloo(tmp_path, world):
    out = str(tmp_path / "gp")
    mp.spawn(_gp_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    total_own = 0
    for r in range(world):
        ok, halo_ok, n_local, n_own, n_halo = np.load("%s.%d.npy" % (out, r))
        assert ok and halo_ok
        assert n_local == n_own + n_halo + (world - 1)
        total_own += n_own
    assert total_own == 72

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

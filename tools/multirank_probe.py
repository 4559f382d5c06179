"""Graph-partitioned mode end to end with several ranks SHARING one GPU (gloo process group, border buffers
staged through the host): exchange counts / bytes and parity at sizes above the unit tests.  Timings are not
scaling numbers (the ranks time-slice one device); the counts are what a multi-GPU run would exchange.

    python tools/multirank_probe.py > profiles/r2_graph_partitioned_gloo.jsonl
"""
import json, os, socket, sys, time
import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, kind, mode, nsrc, groups, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import oracle as O
    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200 import generators as G
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if kind == "road512":
        g = G.road_like(512, 512, keep=0.2, seed=1); part = P.strip_partition(512, 512, world)
    elif kind == "road256":
        g = G.road_like(256, 256, keep=0.2, seed=1); part = P.strip_partition(256, 256, world)
    elif kind == "rmat16":
        g = G.rmat(16, 16, 1); part = P.block_partition(g, world)
    elif kind == "tree":
        g = G.random_connected(200000, 2000, seed=3); part = P.mincut_partition(g, world, seed=0)
    else:
        raise SystemExit(kind)
    import random
    srcs = sorted(random.Random(0).sample(range(g.num_vertices), nsrc))
    cfg = P.RunConfig(sources=srcs, num_gpus=world, gpu_mode="graph-partitioned", mode=mode, partition=part,
                      groups=groups, device=0)
    t0 = time.time()
    res = P.run_bc(g, cfg)
    wall = time.time() - t0
    if rank == 0:
        check = srcs[:: max(1, len(srcs) // 8)][:8]
        cfg2 = P.RunConfig(sources=check, num_gpus=world, gpu_mode="graph-partitioned", mode=mode, partition=part,
                           groups=groups, device=0)
    else:
        check = srcs[:: max(1, len(srcs) // 8)][:8]
        cfg2 = P.RunConfig(sources=check, num_gpus=world, gpu_mode="graph-partitioned", mode=mode, partition=part,
                           groups=groups, device=0)
    res2 = P.run_bc(g, cfg2)
    if rank == 0:
        want, _ = O.brandes_bc(g, check)
        err = float(np.max(np.abs(res2.bc - want) / np.maximum(np.abs(want), 1e-9)))
        st = res.stats
        batches = (nsrc + 32 * groups - 1) // (32 * groups)
        rec = {"graph": kind, "n": g.num_vertices, "m": g.num_edges, "world": world, "mode": mode, "sources": nsrc,
               "groups": groups, "batches": batches, "borders": [int(x) for x in res.borders.counts()],
               "levels": st["levels"], "forward": st["forward"], "sharded_tables": st.get("sharded_tables"),
               "forward_exchanges": st["forward_exchanges"], "backward_levels": st["backward_levels"],
               "backward_exchanges": st["backward_exchanges"], "exchanged_bytes_rank0": st["exchanged_bytes"],
               "refinement_iterations": st["iterations"], "state_vertices_rank0": st["state_vertices"],
               "owned_vertices_rank0": st["owned_vertices"], "table_bytes_rank0": st["table_bytes"],
               "wall_s_ranks_sharing_one_gpu": wall, "bc_rel_vs_oracle_8_sources": err, "parity": bool(err <= 1e-9)}
        with open(out, "a") as fh:
            fh.write(json.dumps(rec) + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "graph_partitioned_gloo.jsonl")
    open(out, "w").close()
    cases = [("road256", "hybir", 4, 128, 4), ("road512", "hybir", 4, 128, 4), ("road512", "bsp-baseline", 4, 128, 4),
             ("rmat16", "bsp-baseline", 4, 256, 4), ("tree", "hybir", 4, 64, 2), ("tree", "bsp-baseline", 4, 64, 2)]
    for kind, mode, world, nsrc, groups in cases:
        mp.spawn(worker, args=(world, free_port(), kind, mode, nsrc, groups, out), nprocs=world, join=True)
    print(open(out).read())

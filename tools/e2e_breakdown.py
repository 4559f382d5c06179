"""Where the end-to-end time of run_bc() goes (host wall clock per stage).

    python tools/e2e_breakdown.py [workload] [sources]

Stages: bc_create (CSR upload + work items), options, bc_run (state allocation
+ kernels + BC copy back), bc_destroy.  `device_ms` is the engine's own CUDA
event time of the kernels inside bc_run.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2008_05718_b200 as P  # noqa: E402
from paper_2008_05718_b200._capi import Engine, MODE_DIRECT  # noqa: E402
from paper_2008_05718_b200.engine import default_groups  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    g, label = bench.workload(name)
    g.pin()
    src = bench.pick_sources(g.num_vertices, k)
    groups = default_groups(g, len(src))
    for rep in range(4):
        t0 = time.perf_counter()
        eng = Engine(g, 0)
        t1 = time.perf_counter()
        eng.set_option("groups", groups)
        eng.set_option("reports", 0)
        t2 = time.perf_counter()
        bc, st = eng.run(src, MODE_DIRECT)
        t3 = time.perf_counter()
        eng.close()
        t4 = time.perf_counter()
        print("rep %d: create %.1f ms, options %.1f ms, run %.1f ms (device %.1f ms), destroy %.1f ms, total %.1f ms"
              % (rep, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, st["ms_total"], (t4 - t3) * 1e3,
                 (t4 - t0) * 1e3), flush=True)
    for rep in range(3):
        t0 = time.perf_counter()
        res = P.run_bc(g, P.RunConfig(sources=src, mode="direct", device=0, per_source_reports=False))
        t1 = time.perf_counter()
        print("run_bc rep %d: %.1f ms (elapsed field %.1f ms)" % (rep, (t1 - t0) * 1e3, res.elapsed * 1e3),
              flush=True)


if __name__ == "__main__":
    main()

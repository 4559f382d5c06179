"""Time the reference's OWN Python implementation on BASELINE config 1 (R-MAT scale-12 EF-8, 2 parts).

Runs in the build container only (it imports /root/reference, which does not exist on the GPU box)
and writes profiles/r2_python_reference_c1.json; bench.py quotes that record beside the C port's
time.  The reference is single-threaded by design, so every figure is one core.

    python tools/time_python_reference.py [oracle_sources] [engine_sources]
"""
import json, os, platform, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
import hybir                                      # the reference package itself
from hybir.oracle import brandes_bc
from paper_2008_05718_b200 import generators as G
import oracle as O

n_oracle = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n_engine = int(sys.argv[2]) if len(sys.argv) > 2 else 24
g = G.rmat(12, 8, 1)
und = g.arc_src < g.arc_dst
edges = [(int(u), int(v), 1) for u, v in zip(g.arc_src[und], g.arc_dst[und])]
rg = hybir.from_edges(g.num_vertices, edges)
assert rg.num_edges == g.num_edges
all_sources = list(range(g.num_vertices))
stride = lambda k: [all_sources[(i * len(all_sources)) // k] for i in range(k)]

sample = stride(n_oracle)
t0 = time.perf_counter()
ref_bc = brandes_bc(rg, sample)
t_oracle = time.perf_counter() - t0
port_bc, _ = O.brandes_bc(g, sample, threads=1)
assert np.allclose(ref_bc.bc, port_bc, rtol=1e-12, atol=1e-12)

rec = {"workload": "BASELINE config 1: R-MAT scale-12 EF-8 seed 1 (n=%d, m=%d), 2 parts" % (g.num_vertices, g.num_edges),
       "where": "build container, %s, 1 core (the reference is single-threaded)" % platform.processor(),
       "oracle_brandes_bc": {"sources": n_oracle, "seconds": t_oracle, "ms_per_source": 1e3 * t_oracle / n_oracle,
                             "teps": g.num_edges * n_oracle / t_oracle,
                             "sample": "every %.0f-th vertex" % (g.num_vertices / n_oracle),
                             "bc_equal_to_c_port": True}}
for mode in ("hybir", "bsp-baseline"):
    srcs = stride(n_engine)
    cfg = hybir.RunConfig(sources=srcs, mode=mode)
    t0 = time.perf_counter()
    res = hybir.run_bc(rg, cfg)
    dt = time.perf_counter() - t0
    want, _ = O.brandes_bc(g, srcs, threads=1)
    rec["run_bc_" + mode] = {"sources": n_engine, "seconds_incl_prepare": dt,
                             "teps_incl_prepare": g.num_edges * n_engine / dt,
                             "reported_mteps": res.mteps,
                             "bc_equal_to_c_port": bool(np.allclose(res.bc, want, rtol=1e-9, atol=1e-12))}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "r2_python_reference_c1.json"), "w") as fh:
    json.dump(rec, fh, indent=1)
print(json.dumps(rec, indent=1))

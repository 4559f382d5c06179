"""Phase times of the end-to-end call of the bench workload (dev tool, run on the GPU box):
python tools/e2e_trace.py  -> wall time of run_bc() and the engine's own phase trace."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G

g = G.rmat(20, 16, 1)
g.pin()
rng = np.random.default_rng(1)
sources = np.sort(rng.choice(g.num_vertices, 1024, replace=False)).tolist()
cfg = P.RunConfig(sources=sources, mode="direct", device=0, per_source_reports=False)
P.run_bc(g, cfg)
for rep in range(3):
    t0 = time.perf_counter()
    res = P.run_bc(g, cfg)
    print("run_bc wall %.2f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
os.environ["BC_B200_TRACE"] = "1"
t0 = time.perf_counter()
res = P.run_bc(g, cfg)
print("traced run_bc wall %.2f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
import cProfile, pstats
del os.environ["BC_B200_TRACE"]
pr = cProfile.Profile(); pr.enable(); P.run_bc(g, cfg); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)

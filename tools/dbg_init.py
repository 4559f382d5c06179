import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_HYBIR
g = G.road_like(40, 40, keep=0.2, seed=5)
srcs = list(range(0, 1600, 37))
with Engine(g) as e:
    e.set_option("groups", 1)
    bc, st = e.run(srcs)
obc, _ = O.brandes_bc(g, srcs)
print("direct ok", np.allclose(bc, obc, rtol=1e-9, atol=1e-12), st["launches"])
part = P.strip_partition(40, 40, 2)
with Engine(g) as e:
    e.set_option("groups", 1); e.set_option("reports", 0)
    e.set_partition(2, part.assignment)
    bc, st = e.run(srcs, MODE_HYBIR)
print("hybir ok", np.allclose(bc, obc, rtol=1e-9, atol=1e-12), st["launches"])

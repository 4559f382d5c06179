import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine
g = G.road_like(80, 80, keep=0.2, seed=5)
srcs = list(range(0, 6400, 61))
obc, _ = O.brandes_bc(g, srcs)
def err(bc): return float(np.max(np.abs(bc - obc) / np.maximum(np.abs(obc), 1e-9)))
for groups in (4, 2, 1):
    for mode in (0, 1, 2):
        for pre_debug in (0, 1):
            with Engine(g) as e:
                e.set_option("groups", groups); e.set_option("deep_compact", mode)
                if pre_debug: e.debug_sources(srcs[:20])
                bc, st = e.run(srcs)
                bc2, _ = e.run(srcs)
            print(dict(groups=groups, mode=mode, pre_debug=pre_debug, err=err(bc), err2=err(bc2), batches=st["batches"], launches=st["launches"]), flush=True)
# per-batch check
for lo in (0, 64):
    sub = srcs[lo:lo + 64]
    ob, _ = O.brandes_bc(g, sub)
    with Engine(g) as e:
        e.set_option("groups", 2); e.set_option("deep_compact", 1)
        bc, st = e.run(sub)
    print("sub", lo, len(sub), float(np.max(np.abs(bc - ob) / np.maximum(np.abs(ob), 1e-9))))

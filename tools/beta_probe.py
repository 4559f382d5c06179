"""push/pull switch thresholds on the renumbered bench graph (dev probe)."""
import os, sys, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine
g = G.rmat(20, 16, 1)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), 1024))
with Engine(g) as e:
    e.set_option("groups", 32); e.set_option("relabel", 1)
    e.run(srcs)
    for beta, late in ((4, 24), (2, 24), (8, 24), (16, 24), (1, 24), (4, 8), (4, 64), (1000000, 24)):
        e.set_option("push_beta", beta); e.set_option("push_beta_late", late)
        e.run(srcs)
        best = min(e.run(srcs)[1]["ms_total"] for _ in range(3))
        st = e.run(srcs)[1]
        print("push_beta %7d late %3d: %.2f ms  (level kernels %.2f ms in %d launches, %d launches in all)" % (
            beta, late, best, st["ms_level"], st["launches_level"], st["launches"]), flush=True)

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_HYBIR, MODE_BSP, MODE_DIRECT
g = G.rmat(12, 8, 1)
p = P.greedy_bipartition(g, 0.5, seed=0)
with Engine(g) as e:
    e.set_option("groups", 4); e.set_option("reports", 0)
    e.set_partition(2, p.assignment)
    srcs = list(range(2944, 2944 + 128))
    d, sg, dl = e.debug_sources(srcs, MODE_HYBIR)
    for i, s in enumerate(srcs):
        od, osg, odl, info = O.brandes_single_source(g, s)
        nd, ns = int((d[i] != od).sum()), int((sg[i] != osg).sum())
        ndl = int((~np.isclose(dl[i], odl, rtol=1e-9, atol=1e-12)).sum())
        if nd or ns or ndl:
            print("src", s, "lane", i % 32, "batch", i // 32, "part", int(p.assignment[s]), "deg", g.degree(s), "bad d/s/dl", nd, ns, ndl, "levels", info["levels"], flush=True)
            bad = np.flatnonzero(sg[i] != osg)[:8]
            print("    sigma at", bad.tolist(), sg[i][bad].tolist(), osg[bad].tolist(), "dist", od[bad].tolist(), "gpu dist", d[i][bad].tolist(), "part", p.assignment[bad].tolist())
    # now with 32-lane batches via run
    for lo in range(2944, 2944 + 128, 32):
        e.set_option("groups", 1)
        bc, _ = e.run(list(range(lo, lo + 32)), MODE_HYBIR)
        obc, _ = O.brandes_bc(g, list(range(lo, lo + 32)))
        print("run 32 from", lo, np.allclose(bc, obc, rtol=1e-9, atol=1e-12))
    for w in (64, 128):
      for lo in range(2944, 2944 + 128, w):
        e.set_option("groups", w // 32)
        bc, _ = e.run(list(range(lo, lo + w)), MODE_HYBIR)
        obc, _ = O.brandes_bc(g, list(range(lo, lo + w)))
        print("run", w, "from", lo, np.allclose(bc, obc, rtol=1e-9, atol=1e-12), "nbad", int((~np.isclose(bc, obc, rtol=1e-9, atol=1e-12)).sum()))

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine
def with_weights(g, seed, wmax):
    rng = np.random.default_rng(seed)
    src, dst = g.arc_src, g.arc_dst
    keep = src < dst
    w = rng.integers(1, wmax + 1, size=int(keep.sum()))
    return P.from_edge_arrays(g.num_vertices, src[keep], dst[keep], w)
g = with_weights(G.random_connected(600, 900, seed=11), 1, 10)
srcs = list(range(0, 600, 7))
for groups in (1, 2, 3):
    for nsrc in (8, 22, 32, 64, 86):
        with Engine(g) as e:
            e.set_option("groups", groups); e.set_option("sssp", 1)
            bc, st = e.run(srcs[:nsrc])
            bc2, st = e.run(srcs[:nsrc])
        obc, info = O.brandes_bc(g, srcs[:nsrc])
        err = np.abs(bc - obc); j = int(err.argmax())
        print(groups, nsrc, "max err %.3e at %d (%.6f vs %.6f) rerun diff %.3e" % (err.max(), j, bc[j], obc[j], np.abs(bc-bc2).max()))
print("---- subsets")
for lo, hi in ((64, 86), (64, 75), (75, 86), (70, 80)):
    sub = srcs[lo:hi]
    with Engine(g) as e:
        e.set_option("groups", 1); e.set_option("sssp", 1)
        bc, st = e.run(sub)
        dist, sigma, delta = e.debug_sources(sub)
    obc, info = O.brandes_bc(g, sub)
    err = np.abs(bc - obc)
    bad = np.nonzero(err > 1e-9)[0]
    print(lo, hi, "bad vertices", bad.tolist()[:10], "err", err[bad][:10])
    tot = np.zeros(g.num_vertices)
    for i, s in enumerate(sub):
        od, osg, odl, _ = O.brandes_single_source(g, int(s))
        d = delta[i].copy(); d[s] = 0
        tot += d
        if not np.allclose(delta[i], odl, rtol=1e-9, atol=1e-12) or not np.array_equal(dist[i], od):
            print("  source", s, "debug mismatch")
    print("   debug-sum vs run max diff", np.abs(tot - bc).max())

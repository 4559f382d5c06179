"""Dev check run on the GPU box: parity on small graphs + first timings."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_2008_05718_b200 import generators as G, from_edges
from paper_2008_05718_b200._capi import Engine

def check(g, sources, tag, groups=4):
    with Engine(g) as e:
        e.set_option("groups", groups)
        d, s, dl = e.debug_sources(sources)
        bc, st = e.run(sources)
    obc, info = O.brandes_bc(g, sources)
    nd = ns = 0; maxrel = 0.0
    for i, src in enumerate(sources):
        od, osg, odl, _ = O.brandes_single_source(g, int(src))
        nd += int((od != d[i]).sum()); ns += int((osg != s[i]).sum())
        den = np.maximum(np.abs(odl), 1e-300)
        rel = np.abs(dl[i] - odl) / den
        rel[odl == 0] = np.abs(dl[i][odl == 0])
        maxrel = max(maxrel, float(rel.max()))
    bcrel = float((np.abs(bc - obc) / np.maximum(np.abs(obc), 1e-12)).max())
    ok = nd == 0 and ns == 0 and maxrel < 1e-9 and bcrel < 1e-9
    print(tag, "OK" if ok else "FAIL", dict(dist_bad=nd, sigma_bad=ns, delta_rel=maxrel, bc_rel=bcrel),
          {k: st[k] for k in ("reached", "arcs_reached", "dag_arcs", "max_levels", "launches")},
          {k: info[k] for k in ("reached", "arcs_reached", "dag_arcs", "max_levels")}, flush=True)
    return ok

ok = True
ok &= check(G.path(4), [0, 1, 2, 3], "p4")
ok &= check(from_edges(4, [(0,1,1),(0,2,1),(1,3,1),(2,3,1)]), [0, 1, 2, 3], "diamond")
ok &= check(G.grid(17, 13), list(range(0, 221, 3)), "grid17x13")
ok &= check(G.random_connected(300, 200, seed=3), list(range(300)), "rc300", groups=3)
g = G.rmat(12, 8, 1)
ok &= check(g, list(range(0, 4096, 7)), "rmat12 subsample")
g14 = G.rmat(14, 16, 1)
ok &= check(g14, list(range(0, 16384, 61)), "rmat14 (hubs)")
print("PARITY", "OK" if ok else "FAIL", flush=True)

if "--time" in sys.argv:
    import random
    t = time.time(); g = G.rmat(20, 16, 1); print("rmat20 build", time.time() - t, g, flush=True)
    srcs = sorted(random.Random(0).sample(range(g.num_vertices), 1024))
    res = []
    for item_arcs in (256, 128, 512):
        for groups in (1, 2, 4, 8):
            with Engine(g) as e:
                e.set_option("groups", groups); e.set_option("item_arcs", item_arcs)
                bc, st = e.run(srcs[:groups * 32])   # warm-up
                t0 = time.time(); bc, st = e.run(srcs); wall = time.time() - t0
            teps = g.num_edges * len(srcs) / (st["ms_total"] / 1e3)
            row = dict(item_arcs=item_arcs, groups=groups, ms=st["ms_total"], fwd=st["ms_forward"], bwd=st["ms_backward"],
                       wall=wall, gteps=teps / 1e9, levels=st["max_levels"], launches=st["launches"])
            print(row, flush=True); res.append(row)
    obc, info = O.brandes_bc(g, srcs[:64])
    with Engine(g) as e:
        bc64, st = e.run(srcs[:64])
    print("rmat20 64-source bc rel", float((np.abs(bc64 - obc) / np.maximum(np.abs(obc), 1e-9)).max()), info, st, flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/first_timing.json", "w"), indent=1)

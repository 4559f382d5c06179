"""Offline: does grouping sources by similarity improve gather utilisation?"""
import sys, random, numpy as np
sys.path.insert(0, '.')
import oracle as O
from paper_2008_05718_b200 import generators as G
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
g = G.rmat(scale, 16, 1)
n = g.num_vertices
deg = np.diff(g.offsets)
cand = [s for s in sorted(random.Random(0).sample(range(n), 1024)) if deg[s] > 0][:256]
Dall = {s: O.brandes_single_source(g, s)[0] for s in cand}
hub = int(np.argmax(deg))
dh = O.brandes_single_source(g, hub)[0]
off, col = g.offsets, g.col_idx
src_of_arc = np.repeat(np.arange(n), deg)
arc_pos = np.arange(len(col)) - off[src_of_arc]
slice_id = np.cumsum(np.r_[0, (deg + 31) // 32])[src_of_arc] + arc_pos // 32
nsl = int(slice_id.max()) + 1

def cost(groups):
    tot_it = 0; tot_pairs = 0; tot_slices = 0
    for grp in groups:
        D = np.stack([Dall[s] for s in grp])
        maxL = D.max()
        for phase in ("fwd", "bwd"):
            for L in range(1, maxL + 1):
                dv = D[:, src_of_arc]; dw = D[:, col]
                hit = (dv == L) & (dw == (L - 1 if phase == "fwd" else L + 1))
                if not hit.any(): continue
                colcnt = np.stack([np.bincount(slice_id, weights=hit[l], minlength=nsl) for l in range(len(grp))])
                maxcol = colcnt.max(axis=0)
                tot_it += np.ceil(maxcol / 4).sum(); tot_pairs += hit.sum(); tot_slices += (maxcol > 0).sum()
    return tot_it, tot_pairs, tot_slices

def report(name, order):
    groups = [order[i:i + 32] for i in range(0, len(order), 32)]
    it, pairs, sl = cost(groups)
    print(f"{name:28s} iterations={it/1e6:.2f}M active slices={sl/1e6:.2f}M pairs={pairs/1e6:.1f}M util={pairs/(it*128):.3f}", flush=True)

report("random (sorted by id)", cand)
report("by dist to top hub, degree", sorted(cand, key=lambda s: (dh[s], -deg[s])))
report("by degree", sorted(cand, key=lambda s: -deg[s]))
ecc = {s: int(Dall[s].max()) for s in cand}
# dense level = level with most vertices
dl = {s: int(np.argmax(np.bincount(Dall[s][Dall[s] >= 0]))) for s in cand}
report("by dense level, then hubdist", sorted(cand, key=lambda s: (dl[s], dh[s], -deg[s])))
# by number of vertices within 2 hops
r2 = {s: int((Dall[s] <= 2).sum() - (Dall[s] < 0).sum()) for s in cand}
report("by |ball(2)|", sorted(cand, key=lambda s: -r2[s]))
nd = {s: int(deg[col[off[s]:off[s+1]]].sum()) for s in cand}
report("by sum of neighbour degrees", sorted(cand, key=lambda s: -nd[s]))
mx = {s: int(deg[col[off[s]:off[s+1]]].max()) for s in cand}
report("by max neighbour degree, nd", sorted(cand, key=lambda s: (-mx[s], -nd[s])))

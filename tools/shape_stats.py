"""Offline (CPU) statistics of the 32x32 hit matrices the level kernels see."""
import sys, random, numpy as np
sys.path.insert(0, '.')
import oracle as O
from paper_2008_05718_b200 import generators as G
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
g = G.rmat(scale, 16, 1)
n = g.num_vertices
srcs = sorted(random.Random(0).sample(range(n), 32))
D = np.stack([O.brandes_single_source(g, s)[0] for s in srcs])  # [32][n]
off, col = g.offsets, g.col_idx
deg = np.diff(off)
src_of_arc = np.repeat(np.arange(n), deg)
maxL = D.max()
print("n", n, "arcs", len(col), "levels", maxL + 1)
for phase in ("fwd", "bwd"):
    for L in range(1, maxL + 1):
        # hit[arc][lane]: fwd: D[lane][v]==L and D[lane][w]==L-1 ; bwd: D[lane][v]==L and D[lane][w]==L+1
        dv = D[:, src_of_arc]; dw = D[:, col]
        hit = (dv == L) & (dw == (L - 1 if phase == "fwd" else L + 1))   # [32][arcs]
        pairs = int(hit.sum())
        if pairs == 0: continue
        # slices: per vertex, chunks of 32 arcs
        arc_pos = np.arange(len(col)) - off[src_of_arc]
        slice_id = off[src_of_arc] // 1 * 0 + (np.cumsum(np.r_[0, (deg + 31) // 32])[src_of_arc] + arc_pos // 32)
        nsl = int(slice_id.max()) + 1
        rowhit = hit.any(axis=0)
        nh = np.bincount(slice_id, weights=rowhit, minlength=nsl)
        colcnt = np.stack([np.bincount(slice_id, weights=hit[l], minlength=nsl) for l in range(32)])  # [32][nsl]
        maxcol = colcnt.max(axis=0); nl = (colcnt > 0).sum(axis=0); tot = colcnt.sum(axis=0)
        act = nh > 0
        it_row = np.ceil(nh[act] / 2).sum(); it_col = np.ceil(maxcol[act] / 4).sum()
        print(f"{phase} L{L}: pairs={pairs/1e6:.2f}M active_slices={act.sum()/1e3:.0f}K of {nsl/1e3:.0f}K  mean nh={nh[act].mean():.1f} nl={nl[act].mean():.1f} maxcol={maxcol[act].mean():.2f} pairs/slice={tot[act].mean():.1f} "
              f"| iters row/2={it_row/1e6:.2f}M col/4={it_col/1e6:.2f}M  util_col={pairs/(it_col*128):.2f}  few-lane(nl<=4) slices {((nl<=4)&act).sum()/act.sum():.2f} holding pairs {tot[(nl<=4)&act].sum()/pairs:.2f}")
        # histogram of maxcol
        h = np.bincount(np.minimum(maxcol[act].astype(int), 33))
        print("    maxcol hist:", {i: int(c) for i, c in enumerate(h) if c})

"""Dev tool: the border-matrix mode on R-MAT graphs of growing size (border tables at scale)."""
import json, os, random, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_DIRECT, MODE_HYBIR, MODE_BSP
for scale in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "14,16").split(",")]:
    g = G.rmat(scale, 16, 1)
    srcs = sorted(random.Random(0).sample(range(g.num_vertices), 256))
    for k in (2, 4):
        part = P.block_partition(g, k)
        with Engine(g) as e:
            e.set_option("reports", 0)
            t0 = time.time(); e.set_partition(k, part.assignment); counts = e.border_counts(k).tolist()
            t1 = time.time(); bc, st = e.run(srcs[:32], MODE_HYBIR); t_tab = time.time() - t1
            bc, st = e.run(srcs, MODE_HYBIR)
            bcb, stb = e.run(srcs, MODE_BSP)
            bcd, std = e.run(srcs, MODE_DIRECT)
        print(json.dumps(dict(scale=scale, k=k, n=g.num_vertices, m=g.num_edges, borders=counts, table_gb=sum(12 * b * b for b in counts) / 1e9,
                              set_partition_s=round(t1 - t0, 2), tables_s=round(t_tab, 2), hybir_ms=round(st["ms_total"], 1),
                              border_ms=round(st["ms_border"], 1), bsp_ms=round(stb["ms_total"], 1), direct_ms=round(std["ms_total"], 1),
                              iterations=st["iterations"],
                              hybir_vs_direct=float(np.max(np.abs(bc - bcd) / np.maximum(np.abs(bcd), 1e-9))),
                              bsp_vs_direct=float(np.max(np.abs(bcb - bcd) / np.maximum(np.abs(bcd), 1e-9))))), flush=True)

import os, random, sys
sys.path.insert(0, "/root/repo")
import paper_2008_05718_b200 as P
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine, MODE_HYBIR
g = G.rmat(16, 16, 1)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), 256))
part = P.block_partition(g, 2)
with Engine(g) as e:
    e.set_option("reports", 0)
    e.set_partition(2, part.assignment)
    bc, st = e.run(srcs, MODE_HYBIR)
print(st["ms_total"], st["ms_border"])

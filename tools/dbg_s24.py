import os, sys, time, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_05718_b200 import generators as G
from paper_2008_05718_b200._capi import Engine
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = G.rmat(scale, 16, 1)
srcs = sorted(random.Random(0).sample(range(g.num_vertices), 256))
with Engine(g) as e:
    e.set_option("groups", 4)
    e.run(srcs[:128])
    for rep in range(3):
        t0 = time.time(); bc, st = e.run(srcs); wall = time.time() - t0
        print(dict(wall_ms=round(wall*1e3,1), ms=round(st["ms_total"],1), fwd=round(st["ms_forward"],1), bwd=round(st["ms_backward"],1), launches=st["launches"]), flush=True)
    os.environ["BC_B200_TRACE"] = "1"
with Engine(g) as e:
    e.set_option("groups", 4)
    e.run(srcs[:128])
    print("---- traced run", flush=True)
    e.run(srcs)

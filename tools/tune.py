"""Dev tool (GPU box): time library variants on the bench workload."""
import glob, json, os, random, subprocess, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def cached_graph(name):
    from paper_2008_05718_b200 import generators as G
    from paper_2008_05718_b200.graph import Graph
    path = "/tmp/%s.npz" % name
    if os.path.exists(path):
        z = np.load(path)
        return Graph(int(z["n"]), int(z["m"]), z["off"], z["col"])
    if name == "er22":
        g = G.erdos_renyi(1 << 22, 1 << 26, 1)
    else:
        scale, ef = {"rmat20": (20, 16), "rmat22": (22, 16), "rmat18": (18, 16)}[name]
        g = G.rmat(scale, ef, 1)
    np.savez(path, n=g.num_vertices, m=g.num_edges, off=g.offsets, col=g.col_idx)
    return g

def child(name, groups_list, item_list, nsrc):
    from paper_2008_05718_b200._capi import Engine
    g = cached_graph(name)
    srcs = sorted(random.Random(0).sample(range(g.num_vertices), nsrc))
    for item_arcs in item_list:
        for groups in groups_list:
            with Engine(g) as e:
                e.set_option("groups", groups); e.set_option("item_arcs", item_arcs)
                e.run(srcs[:groups * 32])
                best = None
                for rep in range(2):
                    bc, st = e.run(srcs)
                    if best is None or st["ms_total"] < best["ms_total"]: best = st
            print(json.dumps(dict(lib=os.path.basename(os.environ.get("BC_B200_LIB", "default")), item_arcs=item_arcs, groups=groups,
                                  ms=round(best["ms_total"], 2), fwd=round(best["ms_forward"], 2), bwd=round(best["ms_backward"], 2),
                                  gteps=round(g.num_edges * nsrc / best["ms_total"] / 1e6, 1), bcsum=float(bc.sum()))), flush=True)

if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(sys.argv[2], json.loads(sys.argv[3]), json.loads(sys.argv[4]), int(sys.argv[5]))
    else:
        name = sys.argv[1]; groups = sys.argv[2]; items = sys.argv[3]; nsrc = sys.argv[4]
        cached_graph(name)
        libs = sorted(glob.glob(os.path.join(ROOT, "paper_2008_05718_b200", "variants", "*.so"))) if len(sys.argv) < 6 else sys.argv[5:]
        for lib in libs:
            env = dict(os.environ)
            if lib != "default": env["BC_B200_LIB"] = lib
            subprocess.run([sys.executable, __file__, "child", name, groups, items, nsrc], env=env)

"""Dev tool (GPU box): the child-driven backward levels (option bwd_push) against the parent-driven
sweep on the bench workload -- device time, forward / backward split, BC agreement, oracle sample.

    python tools/bwd_push_probe.py [workload] [sources] [relabel]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2008_05718_b200._capi import Engine, MODE_DIRECT  # noqa: E402
from paper_2008_05718_b200.engine import default_groups  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    relabel = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    g, label = bench.workload(name)
    src = bench.pick_sources(g.num_vertices, k)
    groups = default_groups(g, len(src))
    ref = None
    for beta in (0, 4, 16):
        with Engine(g, 0) as e:
            e.set_option("groups", groups)
            e.set_option("reports", 0)
            e.set_option("relabel", relabel)
            e.set_option("bwd_push", beta)
            e.run(src, MODE_DIRECT)
            best = None
            for rep in range(3):
                bc, st = e.run(src, MODE_DIRECT)
                if best is None or st["ms_total"] < best["ms_total"]:
                    best = st
        if ref is None:
            ref = bc
        rel = float(np.max(np.abs(bc - ref) / np.maximum(np.abs(ref), 1e-300)))
        print(json.dumps(dict(workload=name, bwd_push=beta, ms=round(best["ms_total"], 3),
                              fwd=round(best["ms_forward"], 3), bwd=round(best["ms_backward"], 3),
                              launches=int(best.get("launches", 0)),
                              gteps=round(g.num_edges * len(src) / best["ms_total"] / 1e6, 1),
                              max_rel_vs_parent_driven=rel)), flush=True)
    # oracle on a strided sample of sources, default option
    import oracle as O
    sample = src[:: max(1, len(src) // 6)][:6]
    want = np.asarray(O.brandes_bc(g, sample)[0])
    with Engine(g, 0) as e:
        e.set_option("reports", 0)
        got, _ = e.run(sample, MODE_DIRECT)
    scale = max(float(np.abs(want).max()), 1.0)
    print(json.dumps(dict(oracle_sample=len(sample), max_abs_over_scale=float(np.max(np.abs(got - want)) / scale))), flush=True)


if __name__ == "__main__":
    main()

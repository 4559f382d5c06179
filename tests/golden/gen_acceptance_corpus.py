"""Generate tests/golden/acceptance_corpus.json by running the REFERENCE package over its own
acceptance corpus (pkg/tests/test_acceptance.py:69-153): 200 seeded graphs (n 6..400, every
second one weighted, split ratio 0.5 / 0.7, 5 sampled sources each, rng = Random(20240817)).

Run in the build container only (it imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_acceptance_corpus.py

Recorded per graph: the generator arguments, the reference's partition assignment, the sources,
``run_bc`` BC in hybir mode (bsp-baseline is asserted equal to 1e-9 here, as the reference's own
acceptance criterion 8 does) and the per-source report counters of both modes.
"""

import json
import os
import random
import sys
import tempfile

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402

import hybir as H  # noqa: E402
from hybir.engine import RunConfig, run_bc  # noqa: E402
from conftest import random_connected_graph  # noqa: E402  (the reference's own factory)

CORPUS_SIZE, SOURCES_PER_GRAPH = 200, 5


def main():
    rng = random.Random(20240817)
    doc = {"generator": "tests/golden/gen_acceptance_corpus.py", "reference": "hybir 0.1.0", "records": []}
    for i in range(CORPUS_SIZE):
        n = rng.randint(6, 12) if i < 40 else 13 + int(387 * rng.random() ** 2)
        weighted = i % 2 == 1
        ratio = 0.5 if i % 3 else 0.7
        extra = rng.randint(0, n)
        g = random_connected_graph(n, extra, weighted=weighted, seed=1000 + i)
        p = H.greedy_bipartition(g, ratio, seed=i, restarts=4)
        sources = rng.sample(range(n), min(SOURCES_PER_GRAPH, n))
        with tempfile.NamedTemporaryFile("w", suffix=".part", delete=False) as fh:
            fh.write("\n".join(str(int(x)) for x in p.assignment) + "\n")
            pfile = fh.name
        res_h = run_bc(g, RunConfig(sources=sources, mode="hybir", partition_file=pfile))
        res_b = run_bc(g, RunConfig(sources=sources, mode="bsp-baseline", partition_file=pfile))
        os.unlink(pfile)
        assert np.allclose(res_h.bc, res_b.bc, rtol=1e-9, atol=1e-12)
        doc["records"].append({
            "i": i, "n": n, "extra": extra, "weighted": weighted, "ratio": ratio, "m": int(g.num_edges),
            "assignment": "".join(str(int(x)) for x in p.assignment), "sources": sources,
            "bc": res_h.bc.tolist(),
            "hybir": [[r["forward"]["iterations"], r["forward"]["comm_events"], *r["forward"]["max_level"],
                       r["backward"]["sync_events"], r["backward"]["comm_bytes"], *r["backward"]["levels"]]
                      for r in res_h.per_source],
            "bsp": [[r["forward"]["supersteps"], r["forward"]["comm_events"], *r["forward"]["max_level"],
                     r["backward"]["sync_events"], r["backward"]["comm_bytes"], *r["backward"]["levels"]]
                    for r in res_b.per_source],
        })
        if i % 20 == 0:
            print(i, n, weighted, flush=True)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "acceptance_corpus.json")
    with open(path, "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

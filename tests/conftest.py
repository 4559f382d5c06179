"""Shared fixtures.  GPU tests carry ``@pytest.mark.gpu`` and call the CUDA
engine through its C ABI; everything else runs on CPU (oracle vs golden
vectors, host logic, library symbols, gloo multi-process)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: full-size configuration, minutes on a B200")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def graph_from_record(rec):
    from paper_2008_05718_b200 import from_edges
    edges = np.asarray(rec["edges"], dtype=np.int64).reshape(-1, 2)
    return from_edges(rec["n"], edges)


@pytest.fixture(scope="session")
def golden_graphs(golden):
    return {rec["name"]: (graph_from_record(rec), rec) for rec in golden["graphs"]}


@pytest.fixture(scope="session")
def rmat12():
    from paper_2008_05718_b200 import generators as G
    return G.rmat(12, 8, 1)

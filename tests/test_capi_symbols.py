"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/bc_b200.h declares; without a device it fails loudly."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2008_05718_b200 import _build, _capi, generators as G
from paper_2008_05718_b200.errors import EngineError


@pytest.fixture(scope="module")
def lib_path():
    return _build.build()


def test_header_and_binding_agree(lib_path):
    header = open(os.path.join(ROOT, "include", "bc_b200.h")).read()
    declared = sorted(set(re.findall(r"\b(bc_[a-z_]+)\s*\(", header)))
    assert declared == sorted(_capi.SYMBOLS)
    L = ctypes.CDLL(lib_path)
    for name in declared:
        assert hasattr(L, name), name


def test_stats_struct_layout_matches_the_header():
    # bc_stats is filled by the library and read through ctypes: same fields, same order, same types
    header = open(os.path.join(ROOT, "include", "bc_b200.h")).read()
    body = re.search(r"typedef struct bc_stats \{(.*?)\} bc_stats;", header, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\b(int64_t|double)\s+([a-z_0-9]+)\s*;", body)
    ctype = {"int64_t": ctypes.c_int64, "double": ctypes.c_double}
    assert [(name, ctype[t]) for t, name in fields] == list(_capi.BcStats._fields_)
    assert ctypes.sizeof(_capi.BcStats) == 8 * len(fields)


def test_library_is_sm100a(lib_path):
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-lelf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; the failure path is for CPU-only hosts")
    with pytest.raises(EngineError, match="no CPU fallback"):
        _capi.Engine(G.path(4))


def test_product_code_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2008_05718_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f

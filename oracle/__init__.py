"""CPU oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes front end of ``oracle/liboracle.so`` (built from ``brandes_oracle.c``
by ``make -C oracle`` or ``__graft_entry__.build()``).  The partitioned
(border-matrix) phases have no port here: they are pinned by golden vectors the
reference itself produced (``tests/golden/``).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; nothing
under ``paper_2008_05718_b200/`` does.

Parity status: pinned -- see ``tests/test_oracle.py`` (reference known-answer
vectors and golden fixtures generated from the reference package itself).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile liboracle.so with the system gcc (OpenMP when available)."""
    so = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "brandes_oracle.c")
    if not force and os.path.exists(so) and os.path.getmtime(so) >= os.path.getmtime(src):
        return so
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    base = [cc, "-O3", "-fPIC", "-std=c11", "-shared", "-o", so, src]
    try:
        subprocess.run(base[:1] + ["-fopenmp"] + base[1:], check=True, capture_output=True)
    except (subprocess.CalledProcessError, FileNotFoundError):
        subprocess.run(base, check=True, capture_output=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        so = build()
        L = ctypes.CDLL(so)
        L.oracle_brandes_single_source.restype = ctypes.c_int
        L.oracle_brandes_single_source.argtypes = [
            ctypes.c_int64, _i64p, _i32p, ctypes.c_int64, _i64p, _f64p, _f64p,
            ctypes.POINTER(ctypes.c_double), _i64p]
        L.oracle_brandes_bc.restype = ctypes.c_int
        L.oracle_brandes_bc.argtypes = [
            ctypes.c_int64, _i64p, _i32p, _i64p, ctypes.c_int64, _f64p, ctypes.c_int,
            _i64p, ctypes.POINTER(ctypes.c_double)]
        L.oracle_brandes_single_source_w.restype = ctypes.c_int
        L.oracle_brandes_single_source_w.argtypes = [
            ctypes.c_int64, _i64p, _i32p, _i64p, ctypes.c_int64, _i64p, _f64p, _f64p,
            ctypes.POINTER(ctypes.c_double), _i64p]
        L.oracle_brandes_bc_w.restype = ctypes.c_int
        L.oracle_brandes_bc_w.argtypes = [
            ctypes.c_int64, _i64p, _i32p, _i64p, _i64p, ctypes.c_int64, _f64p, ctypes.c_int,
            _i64p, ctypes.POINTER(ctypes.c_double)]
        L.oracle_masked_relax.restype = ctypes.c_int
        L.oracle_masked_relax.argtypes = [
            ctypes.c_int64, _i64p, _i32p, ctypes.c_void_p, ctypes.c_int64, _i64p, _i64p, _f64p,
            ctypes.c_int64, _i64p, _f64p]
        _LIB = L
    return _LIB


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def brandes_single_source(g, s: int):
    """(dist, sigma, delta, info): dist int64 with -1 = unreached (oracle.py:29-67)."""
    n = g.num_vertices
    dist = np.empty(n, dtype=np.int64)
    sigma = np.empty(n, dtype=np.float64)
    delta = np.empty(n, dtype=np.float64)
    smax = ctypes.c_double(0.0)
    stats = np.zeros(4, dtype=np.int64)
    if g.unit_weight:
        rc = lib().oracle_brandes_single_source(n, g.offsets, g.col_idx, int(s), dist, sigma, delta,
                                                ctypes.byref(smax), stats)
    else:   # positive integer weights: the reference's heap Dijkstra
        rc = lib().oracle_brandes_single_source_w(n, g.offsets, g.col_idx, g.arc_weight, int(s), dist,
                                                  sigma, delta, ctypes.byref(smax), stats)
    if rc:
        raise ValueError("oracle_brandes_single_source failed with status %d" % rc)
    info = {"reached": int(stats[0]), "levels": int(stats[1]), "arcs_reached": int(stats[2]),
            "dag_arcs": int(stats[3]), "sigma_max": smax.value}
    return dist, sigma, delta, info


def brandes_bc(g, sources=None, threads: int | None = None):
    """(bc, info) over ``sources`` (all vertices when None) (oracle.py:70-82)."""
    n = g.num_vertices
    src = np.arange(n, dtype=np.int64) if sources is None else np.asarray(list(sources), dtype=np.int64)
    bc = np.zeros(n, dtype=np.float64)
    tot = np.zeros(4, dtype=np.int64)
    smax = ctypes.c_double(0.0)
    t = threads or host_threads()
    if g.unit_weight:
        rc = lib().oracle_brandes_bc(n, g.offsets, g.col_idx, src, len(src), bc, int(t), tot,
                                     ctypes.byref(smax))
    else:
        rc = lib().oracle_brandes_bc_w(n, g.offsets, g.col_idx, g.arc_weight, src, len(src), bc, int(t),
                                       tot, ctypes.byref(smax))
    if rc:
        raise ValueError("oracle_brandes_bc failed with status %d" % rc)
    info = {"reached": int(tot[0]), "arcs_reached": int(tot[1]), "dag_arcs": int(tot[2]),
            "max_levels": int(tot[3]), "sigma_max": smax.value, "threads": int(t)}
    return bc, info


def masked_relax(g, mask, seeds):
    """Unit-weight restatement of ``initial_relax`` (relax.py:42-103).

    ``seeds`` is a list of (vertex, dist, sigma_base); returns (dist, sigma)
    with ``g.inf_distance`` where unreached.  Raises ``LookupError`` for a
    seed outside the mask (the reference raises ContractViolation).
    """
    n = g.num_vertices
    sv = np.asarray([x[0] for x in seeds], dtype=np.int64)
    sd = np.asarray([x[1] for x in seeds], dtype=np.int64)
    ss = np.asarray([x[2] for x in seeds], dtype=np.float64)
    dist = np.empty(n, dtype=np.int64)
    sigma = np.empty(n, dtype=np.float64)
    mptr = None
    if mask is not None:
        m8 = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
        mptr = m8.ctypes.data_as(ctypes.c_void_p)
    rc = lib().oracle_masked_relax(n, g.offsets, g.col_idx, mptr, len(sv), sv, sd, ss,
                                   int(g.inf_distance), dist, sigma)
    if rc == 3:
        raise LookupError("active vertex outside worker partition")
    if rc:
        raise ValueError("oracle_masked_relax failed with status %d" % rc)
    return dist, sigma

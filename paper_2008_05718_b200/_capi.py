"""ctypes binding of the C ABI in ``include/bc_b200.h``.

This is the only door from the Python host code to the arithmetic.  If the
shared library is missing or cannot be loaded the import of the *engine*
fails with ``EngineError`` -- there is deliberately no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import EngineError, InputError

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("BC_B200_LIB") or os.path.join(HERE, "libbc_b200.so")  # env: tuning variants

BC_OK, BC_ERR_INTERNAL, BC_ERR_INPUT = 0, 1, 2
BC_UNREACHED = -1
MODE_DIRECT, MODE_HYBIR, MODE_BSP = 0, 1, 2

# Every symbol include/bc_b200.h declares (checked by tests/test_capi_symbols.py).
SYMBOLS = (
    "bc_create", "bc_set_weights", "bc_set_option", "bc_set_partition", "bc_run", "bc_run_device",
    "bc_debug_sources", "bc_get_reports", "bc_get_border_counts", "bc_get_border_tables",
    "bc_get_border_frontier", "bc_set_border_tables",
    "bc_dist_setup", "bc_dist_set_cut_arcs", "bc_dist_plan_backward", "bc_dist_pack", "bc_dist_unpack",
    "bc_dist_unpack_all",
    "bc_dist_get_stats", "bc_dist_begin", "bc_dist_forward_level", "bc_dist_backward_level",
    "bc_dist_export", "bc_dist_import", "bc_dist_get_live", "bc_dist_set_live", "bc_dist_finish",
    "bc_dist_hybir_setup", "bc_dist_hybir_get_table", "bc_dist_hybir_set_table",
    "bc_dist_hybir_seed_count", "bc_dist_hybir_seeds", "bc_dist_hybir_forward", "bc_dist_hybir_set_depth",
    "bc_dist_hybir_shard_tables", "bc_dist_hybir_border_step",
    "bc_last_error", "bc_destroy", "bc_release_cached_memory",
)


class BcStats(ctypes.Structure):
    _fields_ = [
        ("sources", ctypes.c_int64), ("batches", ctypes.c_int64), ("max_levels", ctypes.c_int64),
        ("reached", ctypes.c_int64), ("arcs_reached", ctypes.c_int64), ("dag_arcs", ctypes.c_int64),
        ("launches", ctypes.c_int64), ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
        ("ms_total", ctypes.c_double), ("ms_forward", ctypes.c_double),
        ("ms_backward", ctypes.c_double), ("ms_border", ctypes.c_double),
        ("iterations", ctypes.c_int64), ("comm_events", ctypes.c_int64),
        ("sync_events", ctypes.c_int64), ("comm_bytes", ctypes.c_int64),
        ("launches_forward", ctypes.c_int64), ("launches_backward", ctypes.c_int64),
        ("launches_level", ctypes.c_int64),
        ("ms_level", ctypes.c_double), ("launches_level_timed", ctypes.c_int64),
        ("level_scan_arcs", ctypes.c_int64), ("level_pairs", ctypes.c_int64),
        ("level_vertex_lanes", ctypes.c_int64), ("level_dense_words", ctypes.c_int64),
        ("level_entries", ctypes.c_int64), ("level_model_bytes", ctypes.c_int64),
        ("lookahead_batches", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load():
    """Load libbc_b200.so (once) and declare the prototypes."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise EngineError(
            "CUDA engine library %s is missing; build it with "
            "`python -m paper_2008_05718_b200._build` (there is no CPU fallback)" % SO_PATH)
    try:
        L = ctypes.CDLL(SO_PATH)
    except OSError as exc:  # pragma: no cover - depends on the machine
        raise EngineError("cannot load %s: %s" % (SO_PATH, exc)) from exc
    vp, i64, i32, cint = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
    L.bc_create.restype = cint
    L.bc_create.argtypes = [i64, i64, vp, vp, cint, ctypes.POINTER(vp)]
    L.bc_set_weights.restype = cint
    L.bc_set_weights.argtypes = [vp, vp]
    L.bc_set_option.restype = cint
    L.bc_set_option.argtypes = [vp, ctypes.c_char_p, i64]
    L.bc_set_partition.restype = cint
    L.bc_set_partition.argtypes = [vp, cint, vp]
    L.bc_run.restype = cint
    L.bc_run.argtypes = [vp, cint, vp, i64, vp, ctypes.POINTER(BcStats)]
    L.bc_run_device.restype = cint
    L.bc_run_device.argtypes = [vp, cint, vp, i64, vp, vp, ctypes.POINTER(BcStats)]
    L.bc_debug_sources.restype = cint
    L.bc_debug_sources.argtypes = [vp, cint, vp, i64, vp, vp, vp]
    L.bc_get_reports.restype = cint
    L.bc_get_reports.argtypes = [vp, vp, i64]
    L.bc_get_border_counts.restype = cint
    L.bc_get_border_counts.argtypes = [vp, vp]
    L.bc_get_border_tables.restype = cint
    L.bc_get_border_tables.argtypes = [vp, cint, vp, vp, vp]
    L.bc_set_border_tables.restype = cint
    L.bc_set_border_tables.argtypes = [vp, cint, vp, vp]
    L.bc_get_border_frontier.restype = cint
    L.bc_get_border_frontier.argtypes = [vp, i64, vp, vp, vp]
    L.bc_dist_setup.restype = cint
    L.bc_dist_setup.argtypes = [vp, cint, cint, vp, vp, vp]
    L.bc_dist_set_cut_arcs.restype = cint
    L.bc_dist_set_cut_arcs.argtypes = [vp, vp, vp]
    L.bc_dist_plan_backward.restype = cint
    L.bc_dist_plan_backward.argtypes = [vp, cint, vp, vp]
    L.bc_dist_pack.restype = cint
    L.bc_dist_pack.argtypes = [vp, cint, vp, i64, i64, vp]
    L.bc_dist_unpack.restype = cint
    L.bc_dist_unpack.argtypes = [vp, cint, cint, vp, i64, i64, i64, vp]
    L.bc_dist_unpack_all.restype = cint
    L.bc_dist_unpack_all.argtypes = [vp, cint, vp, i64, i64, i64, vp, cint, vp]
    L.bc_dist_get_stats.restype = cint
    L.bc_dist_get_stats.argtypes = [vp, ctypes.POINTER(BcStats)]
    L.bc_dist_begin.restype = cint
    L.bc_dist_begin.argtypes = [vp, vp, i64, vp]
    L.bc_dist_forward_level.restype = cint
    L.bc_dist_forward_level.argtypes = [vp, cint, vp]
    L.bc_dist_backward_level.restype = cint
    L.bc_dist_backward_level.argtypes = [vp, cint, cint, vp]
    L.bc_dist_export.restype = cint
    L.bc_dist_export.argtypes = [vp, cint, cint, vp, vp, i64, ctypes.POINTER(i64), vp]
    L.bc_dist_import.restype = cint
    L.bc_dist_import.argtypes = [vp, cint, cint, cint, vp, vp, vp]
    L.bc_dist_get_live.restype = cint
    L.bc_dist_get_live.argtypes = [vp, cint, vp, vp]
    L.bc_dist_set_live.restype = cint
    L.bc_dist_set_live.argtypes = [vp, cint, vp, vp]
    L.bc_dist_finish.restype = cint
    L.bc_dist_finish.argtypes = [vp, vp, vp]
    L.bc_dist_hybir_setup.restype = cint
    L.bc_dist_hybir_setup.argtypes = [vp, vp, vp, vp]
    L.bc_dist_hybir_get_table.restype = cint
    L.bc_dist_hybir_get_table.argtypes = [vp, cint, vp, vp]
    L.bc_dist_hybir_set_table.restype = cint
    L.bc_dist_hybir_set_table.argtypes = [vp, cint, vp, vp]
    L.bc_dist_hybir_seed_count.restype = i64
    L.bc_dist_hybir_seed_count.argtypes = [vp]
    L.bc_dist_hybir_seeds.restype = cint
    L.bc_dist_hybir_seeds.argtypes = [vp, vp, vp, i64, vp, vp, vp]
    L.bc_dist_hybir_forward.restype = cint
    L.bc_dist_hybir_forward.argtypes = [vp, vp, vp, ctypes.POINTER(cint), ctypes.POINTER(i64), vp]
    L.bc_dist_hybir_shard_tables.restype = cint
    L.bc_dist_hybir_shard_tables.argtypes = [vp]
    L.bc_dist_hybir_border_step.restype = cint
    L.bc_dist_hybir_border_step.argtypes = [vp, cint, vp, vp, vp, vp, ctypes.POINTER(cint), vp]
    L.bc_dist_hybir_set_depth.restype = cint
    L.bc_dist_hybir_set_depth.argtypes = [vp, cint, vp]
    L.bc_last_error.restype = ctypes.c_char_p
    L.bc_last_error.argtypes = [vp]
    L.bc_destroy.restype = None
    L.bc_destroy.argtypes = [vp]
    L.bc_release_cached_memory.restype = None
    L.bc_release_cached_memory.argtypes = []
    _lib = L
    return L


def release_cached_memory():
    """Return the device blocks cached by closed engines to the CUDA driver."""
    load().bc_release_cached_memory()


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Engine:
    """Owns one ``bc_handle`` (one CUDA device, one host thread)."""

    def __init__(self, g, device: int = 0):
        self._lib = load()
        self._h = ctypes.c_void_p()
        self.n = g.num_vertices
        self.graph = g
        off = np.ascontiguousarray(g.offsets, dtype=np.int64)
        col = np.ascontiguousarray(g.col_idx, dtype=np.int32)
        rc = self._lib.bc_create(self.n, len(col), _ptr(off), _ptr(col), int(device),
                                 ctypes.byref(self._h))
        if rc != BC_OK:
            self._h = ctypes.c_void_p()
            self._raise(rc, handle=None)
        self.h2d_bytes_graph = off.nbytes + col.nbytes
        if not g.unit_weight:
            w = np.ascontiguousarray(g.arc_weight, dtype=np.int64)
            if len(w) and (w.max() >= 2 ** 31 or w.min() < 1):
                self.close()
                raise InputError("arc weights must be integers in [1, 2^31) on the GPU path")
            w32 = w.astype(np.int32)
            rc = self._lib.bc_set_weights(self._h, _ptr(w32))
            if rc != BC_OK:
                self._raise(rc)
            self.h2d_bytes_graph += w32.nbytes

    # -- plumbing ---------------------------------------------------------
    def _raise(self, rc, handle="self"):
        h = self._h if handle == "self" else None
        msg = self._lib.bc_last_error(h)
        msg = msg.decode() if msg else "status %d" % rc
        raise (InputError if rc == BC_ERR_INPUT else EngineError)(msg)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.bc_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- API ----------------------------------------------------------------
    def set_option(self, key: str, value: int):
        rc = self._lib.bc_set_option(self._h, key.encode(), int(value))
        if rc != BC_OK:
            self._raise(rc)

    def set_partition(self, k: int, assignment):
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        if len(a) != self.n:
            raise InputError("partition assignment has %d entries, graph has %d vertices"
                             % (len(a), self.n))
        rc = self._lib.bc_set_partition(self._h, int(k), _ptr(a))
        if rc != BC_OK:
            self._raise(rc)

    def run(self, sources, mode: int = MODE_DIRECT):
        """Host buffers in, host BC vector out: (bc float64[n], stats dict)."""
        src = np.ascontiguousarray(sources, dtype=np.int64)
        bc = np.empty(self.n, dtype=np.float64)     # bc_run overwrites all n entries
        st = BcStats()
        rc = self._lib.bc_run(self._h, int(mode), _ptr(src), len(src), _ptr(bc), ctypes.byref(st))
        if rc != BC_OK:
            self._raise(rc)
        return bc, st.as_dict()

    def run_device(self, sources, bc_dev_ptr: int, stream_ptr: int = 0, mode: int = MODE_DIRECT):
        """Accumulate into a device vector (raw pointer) on the given CUDA stream."""
        src = np.ascontiguousarray(sources, dtype=np.int64)
        st = BcStats()
        rc = self._lib.bc_run_device(self._h, int(mode), _ptr(src), len(src),
                                     ctypes.c_void_p(bc_dev_ptr),
                                     ctypes.c_void_p(stream_ptr) if stream_ptr else None,
                                     ctypes.byref(st))
        if rc != BC_OK:
            self._raise(rc)
        return st.as_dict()

    def debug_sources(self, sources, mode: int = MODE_DIRECT, want=("dist", "sigma", "delta")):
        """Per-source (dist int32[k,n], sigma f64[k,n], delta f64[k,n]); -1 = unreached."""
        src = np.ascontiguousarray(sources, dtype=np.int64)
        k = len(src)
        dist = np.empty((k, self.n), dtype=np.int32) if "dist" in want else None
        sigma = np.empty((k, self.n), dtype=np.float64) if "sigma" in want else None
        delta = np.empty((k, self.n), dtype=np.float64) if "delta" in want else None
        rc = self._lib.bc_debug_sources(self._h, int(mode), _ptr(src), k, _ptr(dist), _ptr(sigma),
                                        _ptr(delta))
        if rc != BC_OK:
            self._raise(rc)
        return dist, sigma, delta

    def reports(self, n_sources: int):
        out = np.zeros((n_sources, 8), dtype=np.int64)
        rc = self._lib.bc_get_reports(self._h, _ptr(out), n_sources)
        if rc != BC_OK:
            self._raise(rc)
        return out

    def border_counts(self, k: int):
        out = np.zeros(k, dtype=np.int64)
        rc = self._lib.bc_get_border_counts(self._h, _ptr(out))
        if rc != BC_OK:
            self._raise(rc)
        return out

    def border_tables(self, part: int, b: int):
        borders = np.zeros(b, dtype=np.int32)
        bm = np.zeros((b, b), dtype=np.int32)
        sm = np.zeros((b, b), dtype=np.float64)
        rc = self._lib.bc_get_border_tables(self._h, int(part), _ptr(borders), _ptr(bm), _ptr(sm))
        if rc != BC_OK:
            self._raise(rc)
        return borders, bm, sm

    def set_border_tables(self, part: int, bm, sm):
        """Install the border table of one part from host arrays (a cache hit): bm int32 with
        -1 = unreachable, sm float64, both b_p x b_p."""
        bm = np.ascontiguousarray(bm, dtype=np.int32)
        sm = np.ascontiguousarray(sm, dtype=np.float64)
        if bm.shape != sm.shape or bm.ndim != 2 or bm.shape[0] != bm.shape[1]:
            raise InputError("border tables must be square and of equal shape")
        rc = self._lib.bc_set_border_tables(self._h, int(part), _ptr(bm), _ptr(sm))
        if rc != BC_OK:
            self._raise(rc)

    def border_frontier(self, n_lanes: int, total_borders: int):
        """(dist, sigma, arrival) of the last hybir batch, each [B, n_lanes]."""
        d = np.zeros((total_borders, n_lanes), dtype=np.int32)
        s = np.zeros((total_borders, n_lanes), dtype=np.float64)
        a = np.zeros((total_borders, n_lanes), dtype=np.float64)
        rc = self._lib.bc_get_border_frontier(self._h, n_lanes, _ptr(d), _ptr(s), _ptr(a))
        if rc != BC_OK:
            self._raise(rc)
        return d, s, a

    # -- graph-partitioned multi-GPU mode (device pointers are raw ints) ----
    def _ck(self, rc):
        if rc != BC_OK:
            self._raise(rc)

    def dist_setup(self, rank, world, assignment, border_off, border_v):
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        bo = np.ascontiguousarray(border_off, dtype=np.int64)
        bv = np.ascontiguousarray(border_v, dtype=np.int32)
        self._ck(self._lib.bc_dist_setup(self._h, int(rank), int(world), _ptr(a), _ptr(bo), _ptr(bv)))

    def dist_begin(self, sources, stream=0):
        src = np.ascontiguousarray(sources, dtype=np.int64)
        self._ck(self._lib.bc_dist_begin(self._h, _ptr(src), len(src), ctypes.c_void_p(stream or None)))

    def dist_forward_level(self, level, stream=0):
        self._ck(self._lib.bc_dist_forward_level(self._h, int(level), ctypes.c_void_p(stream or None)))

    def dist_backward_level(self, level, deepest, stream=0):
        self._ck(self._lib.bc_dist_backward_level(self._h, int(level), int(bool(deepest)),
                                                  ctypes.c_void_p(stream or None)))

    def dist_export(self, level, what, masks_ptr, values_ptr, capacity, stream=0) -> int:
        count = ctypes.c_int64(0)
        self._ck(self._lib.bc_dist_export(self._h, int(level), int(what), ctypes.c_void_p(masks_ptr),
                                          ctypes.c_void_p(values_ptr or None), int(capacity),
                                          ctypes.byref(count), ctypes.c_void_p(stream or None)))
        return count.value

    def dist_import(self, level, what, peer, masks_ptr, values_ptr, stream=0):
        self._ck(self._lib.bc_dist_import(self._h, int(level), int(what), int(peer),
                                          ctypes.c_void_p(masks_ptr), ctypes.c_void_p(values_ptr or None),
                                          ctypes.c_void_p(stream or None)))

    def dist_get_live(self, level, groups, stream=0):
        out = np.zeros(groups, dtype=np.uint32)
        self._ck(self._lib.bc_dist_get_live(self._h, int(level), _ptr(out), ctypes.c_void_p(stream or None)))
        return out

    def dist_set_live(self, level, live, stream=0):
        a = np.ascontiguousarray(live, dtype=np.uint32)
        self._ck(self._lib.bc_dist_set_live(self._h, int(level), _ptr(a), ctypes.c_void_p(stream or None)))

    def dist_hybir_setup(self, cin_off, cin_src, cin_w=None):
        co = np.ascontiguousarray(cin_off, dtype=np.int64)
        cs = np.ascontiguousarray(cin_src, dtype=np.int32)
        cw = None if cin_w is None else np.ascontiguousarray(cin_w, dtype=np.int32)
        self._ck(self._lib.bc_dist_hybir_setup(self._h, _ptr(co), _ptr(cs), _ptr(cw)))

    def dist_hybir_get_table(self, part, bm_ptr, sm_ptr):
        self._ck(self._lib.bc_dist_hybir_get_table(self._h, int(part), ctypes.c_void_p(bm_ptr),
                                                   ctypes.c_void_p(sm_ptr)))

    def dist_hybir_set_table(self, part, bm_ptr, sm_ptr):
        self._ck(self._lib.bc_dist_hybir_set_table(self._h, int(part), ctypes.c_void_p(bm_ptr),
                                                   ctypes.c_void_p(sm_ptr)))

    def dist_hybir_seed_count(self) -> int:
        return int(self._lib.bc_dist_hybir_seed_count(self._h))

    def dist_hybir_seeds(self, sources, source_part, seed_dist_ptr, seed_sigma_ptr, stream=0):
        src = np.ascontiguousarray(sources, dtype=np.int64)
        sp = np.ascontiguousarray(source_part, dtype=np.int32)
        self._ck(self._lib.bc_dist_hybir_seeds(self._h, _ptr(src), _ptr(sp), len(src),
                                               ctypes.c_void_p(seed_dist_ptr), ctypes.c_void_p(seed_sigma_ptr),
                                               ctypes.c_void_p(stream or None)))

    def dist_set_cut_arcs(self, cut_off, cut_dst):
        co = np.ascontiguousarray(cut_off, dtype=np.int64)
        cd = np.ascontiguousarray(cut_dst, dtype=np.int32)
        self._ck(self._lib.bc_dist_set_cut_arcs(self._h, _ptr(co), _ptr(cd)))

    def dist_plan_backward(self, depth, stream=0):
        """(entries, values) per level this rank has to publish on the way back: int64[depth, 2]."""
        out = np.zeros((int(depth), 2), dtype=np.int64)
        self._ck(self._lib.bc_dist_plan_backward(self._h, int(depth), _ptr(out), ctypes.c_void_p(stream or None)))
        return out

    def dist_pack(self, level, send_ptr, cap_entries, cap_values, stream=0):
        self._ck(self._lib.bc_dist_pack(self._h, int(level), ctypes.c_void_p(send_ptr), int(cap_entries),
                                        int(cap_values), ctypes.c_void_p(stream or None)))

    def dist_unpack(self, level, peer, recv_ptr, cap_entries, cap_values, n_entries, stream=0):
        self._ck(self._lib.bc_dist_unpack(self._h, int(level), int(peer), ctypes.c_void_p(recv_ptr),
                                          int(cap_entries), int(cap_values), int(n_entries),
                                          ctypes.c_void_p(stream or None)))

    def dist_unpack_all(self, level, recv_ptr, words_per_rank, cap_entries, cap_values, plan_ptr, depth, stream=0):
        self._ck(self._lib.bc_dist_unpack_all(self._h, int(level), ctypes.c_void_p(recv_ptr), int(words_per_rank),
                                              int(cap_entries), int(cap_values), ctypes.c_void_p(plan_ptr),
                                              int(depth), ctypes.c_void_p(stream or None)))

    def dist_stats(self) -> dict:
        st = BcStats()
        self._ck(self._lib.bc_dist_get_stats(self._h, ctypes.byref(st)))
        return st.as_dict()

    def dist_hybir_forward(self, seed_dist_ptr, seed_sigma_ptr, stream=0):
        depth, iters = ctypes.c_int(0), ctypes.c_int64(0)
        self._ck(self._lib.bc_dist_hybir_forward(self._h, ctypes.c_void_p(seed_dist_ptr),
                                                 ctypes.c_void_p(seed_sigma_ptr), ctypes.byref(depth),
                                                 ctypes.byref(iters), ctypes.c_void_p(stream or None)))
        return depth.value, iters.value

    def dist_hybir_shard_tables(self):
        self._ck(self._lib.bc_dist_hybir_shard_tables(self._h))

    def dist_hybir_border_step(self, step, values_ptr=0, flags_ptr=0, seed_dist_ptr=0, seed_sigma_ptr=0,
                               want_flag=False, stream=0):
        """One step of the sharded-table border phase; returns the step's flag (or None)."""
        flag = ctypes.c_int(0)
        self._ck(self._lib.bc_dist_hybir_border_step(
            self._h, int(step), ctypes.c_void_p(values_ptr or None), ctypes.c_void_p(flags_ptr or None),
            ctypes.c_void_p(seed_dist_ptr or None), ctypes.c_void_p(seed_sigma_ptr or None),
            ctypes.byref(flag) if want_flag else None, ctypes.c_void_p(stream or None)))
        return flag.value if want_flag else None

    def dist_hybir_set_depth(self, depth, stream=0):
        self._ck(self._lib.bc_dist_hybir_set_depth(self._h, int(depth), ctypes.c_void_p(stream or None)))

    def dist_finish(self, bc_dev_ptr, stream=0):
        self._ck(self._lib.bc_dist_finish(self._h, ctypes.c_void_p(bc_dev_ptr), ctypes.c_void_p(stream or None)))

"""ctypes bindings of the CPU checkers (TEST / BASELINE INFRASTRUCTURE ONLY).

* ``port()``  -- oracle/libpdb_oracle.so, the C restatement in pdb_oracle.c
* ``ref()``   -- oracle/_ref/libpdb_ref.so, the reference sources themselves
                 (None where they were never built)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "libpdb_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libpdb_ref.so")

_port = None
_ref = None


class OrcPairs(C.Structure):
    _fields_ = [("count", C.c_int64), ("left", C.POINTER(C.c_int32)),
                ("right", C.POINTER(C.c_int32)), ("dist", C.POINTER(C.c_double))]


def _p(a):
    return a.ctypes.data


def port():
    global _port
    if _port is None:
        L = C.CDLL(PORT_PATH)
        i64, i32, f64, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        L.orc_featurize_tiles.argtypes = [vp, i64, i32, i32, i32, i32, i32, i32, vp]
        L.orc_color_histogram_f32.argtypes = [vp, i64, i32, i32, i32, i32, vp]
        L.orc_euclidean.argtypes = [vp, vp, i64]
        L.orc_euclidean.restype = f64
        L.orc_sim_join.argtypes = [vp, i64, vp, i64, i64, f64, i32, i64, i64, i32,
                                   C.POINTER(OrcPairs)]
        L.orc_pairs_free.argtypes = [C.POINTER(OrcPairs)]
        L.orc_pairs_free.restype = None
        L.orc_sim_join_count.argtypes = [vp, i64, vp, i64, i64, f64, i32, i64, i64]
        L.orc_sim_join_count.restype = i64
        L.orc_hist_dim.argtypes = [C.c_int, C.c_int]
        L.orc_cosine_join_bf16.argtypes = [vp, i64, vp, i64, i64, f64, i32, i64, i64, i32,
                                           C.POINTER(OrcPairs)]
        L.orc_cosine_bf16.argtypes = [vp, vp, i64]
        L.orc_cosine_bf16.restype = f64
        L.orc_sim_join_rows.argtypes = [vp, i64, vp, i64, i64, f64, i32, vp, i64, i32,
                                        C.POINTER(OrcPairs)]
        L.orc_sim_join_pruned.argtypes = [vp, i64, vp, i64, i64, f64, i32, i32,
                                          C.POINTER(OrcPairs)]
        L.orc_dedup.argtypes = [vp, i64, i64, f64, vp]
        L.orc_dedup.restype = i64
        _port = L
    return _port


def ref():
    """The reference compiled from its own sources, or None if not built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            return None
        L = C.CDLL(REF_PATH)
        i64, i32, f64, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_featurize_tiles.argtypes = [vp, i64, i32, i32, i32, i32, i32, vp, i32]
        L.ref_color_histogram_f32.argtypes = [vp, i64, i32, i32, i32, vp]
        L.ref_euclidean.argtypes = [vp, vp, i64]
        L.ref_euclidean.restype = f64
        L.ref_sim_join.argtypes = [vp, i64, vp, i64, i32, f64, i32, C.POINTER(i64),
                                   C.POINTER(C.POINTER(i32)), C.POINTER(C.POINTER(i32)),
                                   C.POINTER(C.c_uint64)]
        L.ref_free.argtypes = [vp]
        L.ref_free.restype = None
        L.ref_join_probe_timed.argtypes = [vp, i64, vp, i64, i32, f64, i32, i64, i64, i32,
                                           C.POINTER(f64), C.POINTER(f64)]
        L.ref_join_probe_timed.restype = i64
        L.ref_join_probe_pairs.argtypes = [vp, i64, vp, i64, i32, f64, i32,
                                           C.POINTER(C.POINTER(i32)), C.POINTER(C.POINTER(i32)),
                                           C.POINTER(f64), C.POINTER(f64)]
        L.ref_join_probe_pairs.restype = i64
        L.ref_dedup.argtypes = [vp, i64, i32, f64, vp, C.POINTER(i64)]
        L.ref_dedup_stream.argtypes = [vp, i64, i32, f64, vp]
        L.ref_dedup_stream.restype = i64
        pp = C.POINTER(C.POINTER(i32))
        L.ref_nl_within.argtypes = [vp, i64, vp, i64, i32, f64, C.POINTER(i64), pp, pp]
        L.ref_q1.argtypes = [vp, i64, i32, i32, i32, f64, C.POINTER(i64), pp, pp]
        L.ref_store_write.argtypes = [vp, i64, i32, i32, i32, i32, i32, C.c_char_p]
        L.ref_store_scan.argtypes = [C.c_char_p, i64, i64, vp]
        L.ref_store_scan.restype = i64
        L.ref_run_query.argtypes = [C.c_char_p, i32, i64]
        L.ref_run_query.restype = vp
        _ref = L
    return _ref


# ---- restatement (port) ------------------------------------------------------

def featurize_tiles(frames: np.ndarray, th: int, tw: int, bins: int, mode: int) -> np.ndarray:
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    F, H, W = frames.shape[:3]
    D = port().orc_hist_dim(bins, mode)
    out = np.empty((F * (H // th) * (W // tw), max(D, 1)), dtype=np.float32)
    rc = port().orc_featurize_tiles(_p(frames), F, H, W, th, tw, bins, mode, _p(out))
    if rc:
        raise RuntimeError(f"oracle featurize failed: {rc}")
    return out


def color_histogram(px: np.ndarray, bins: int, mode: int) -> np.ndarray:
    px = np.ascontiguousarray(px, dtype=np.float32)
    n, h, w = px.shape[:3]
    D = port().orc_hist_dim(bins, mode)
    out = np.empty((n, max(D, 1)), dtype=np.float32)
    rc = port().orc_color_histogram_f32(_p(px), n, h, w, bins, mode, _p(out))
    if rc:
        raise RuntimeError(f"oracle histogram failed: {rc}")
    return out


def euclidean(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return port().orc_euclidean(_p(a), _p(b), a.shape[0])


def sim_join(L: np.ndarray, R, tau: float, self_join: bool = False, rows=(0, -1),
             threads: int | None = None):
    """Brute-force pairs sorted by (i, j): (left int32, right int32, dist f64)."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    R = L if self_join else np.ascontiguousarray(R, dtype=np.float32)
    out = OrcPairs()
    th = threads or max(1, os.cpu_count() or 1)
    rc = port().orc_sim_join(_p(L), L.shape[0], _p(R), R.shape[0], L.shape[1], float(tau),
                             int(self_join), rows[0], rows[1], th, C.byref(out))
    if rc:
        raise RuntimeError(f"oracle join failed: {rc}")
    n = out.count
    try:
        if n:
            res = (np.ctypeslib.as_array(out.left, (n,)).copy(),
                   np.ctypeslib.as_array(out.right, (n,)).copy(),
                   np.ctypeslib.as_array(out.dist, (n,)).copy())
        else:
            res = (np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.float64))
    finally:
        port().orc_pairs_free(C.byref(out))
    return res


def _take(out):
    n = out.count
    try:
        if n:
            res = (np.ctypeslib.as_array(out.left, (n,)).copy(),
                   np.ctypeslib.as_array(out.right, (n,)).copy(),
                   np.ctypeslib.as_array(out.dist, (n,)).copy())
        else:
            res = (np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.float64))
    finally:
        port().orc_pairs_free(C.byref(out))
    return res


def sim_join_rows(L: np.ndarray, R, tau: float, rows, self_join: bool = False,
                  threads: int | None = None):
    """Brute force over a list of L rows (ascending, deduplicated here):
    every (i, j) with euclidean <= tau for i in rows (j > i for self joins),
    sorted by (i, j).  Exact early abandon only (pdb_oracle.c (1))."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    R = L if self_join else np.ascontiguousarray(R, dtype=np.float32)
    rows = np.unique(np.asarray(rows, dtype=np.int64))
    out = OrcPairs()
    th = threads or max(1, os.cpu_count() or 1)
    rc = port().orc_sim_join_rows(_p(L), L.shape[0], _p(R), R.shape[0], L.shape[1], float(tau),
                                  int(self_join), _p(rows), rows.shape[0], th, C.byref(out))
    if rc:
        raise RuntimeError(f"oracle join failed: {rc}")
    return _take(out)


def sim_join_pruned(L: np.ndarray, R, tau: float, self_join: bool = False,
                    threads: int | None = None):
    """The full join, all rows, with exact coordinate-window pruning
    (pdb_oracle.c (2)); same result as sim_join()."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    R = L if self_join else np.ascontiguousarray(R, dtype=np.float32)
    out = OrcPairs()
    th = threads or max(1, os.cpu_count() or 1)
    rc = port().orc_sim_join_pruned(_p(L), L.shape[0], _p(R), R.shape[0], L.shape[1],
                                    float(tau), int(self_join), th, C.byref(out))
    if rc:
        raise RuntimeError(f"oracle join failed: {rc}")
    return _take(out)


def cosine_join_bf16(L: np.ndarray, R, min_cos: float, self_join: bool = False, rows=(0, -1),
                     threads: int | None = None):
    """RESTATED cosine join over bf16 bit patterns (uint16 [n, d]): pairs
    sorted by (i, j) with cos >= min_cos: (left, right, cos f64)."""
    L = np.ascontiguousarray(L, dtype=np.uint16)
    R = L if self_join else np.ascontiguousarray(R, dtype=np.uint16)
    out = OrcPairs()
    th = threads or max(1, os.cpu_count() or 1)
    rc = port().orc_cosine_join_bf16(_p(L), L.shape[0], _p(R), R.shape[0], L.shape[1],
                                     float(min_cos), int(self_join), rows[0], rows[1], th,
                                     C.byref(out))
    if rc:
        raise RuntimeError(f"oracle cosine join failed: {rc}")
    n = out.count
    try:
        if n:
            res = (np.ctypeslib.as_array(out.left, (n,)).copy(),
                   np.ctypeslib.as_array(out.right, (n,)).copy(),
                   np.ctypeslib.as_array(out.dist, (n,)).copy())
        else:
            res = (np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.float64))
    finally:
        port().orc_pairs_free(C.byref(out))
    return res


def cosine_bf16(a: np.ndarray, b: np.ndarray) -> float:
    """Restated fp64 cosine of two bf16 rows (uint16 bit patterns)."""
    a = np.ascontiguousarray(a, dtype=np.uint16)
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return port().orc_cosine_bf16(_p(a), _p(b), a.shape[0])


def dedup(X: np.ndarray, tau: float):
    """Restated run_dedup (src/query.cpp:535-566): (rep_of int64 [n],
    n_reps); rep_of[i] is the index of item i's representative."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n = X.shape[0]
    rep_of = np.empty(max(n, 1), dtype=np.int64)
    nr = port().orc_dedup(_p(X), n, X.shape[1] if X.ndim == 2 else 0, float(tau), _p(rep_of))
    if nr < 0:
        raise ValueError("dedup needs tau >= 0")
    return rep_of[:n], int(nr)


# ---- the reference itself ------------------------------------------------------

def ref_featurize_tiles(frames: np.ndarray, th: int, tw: int, bins: int, threads: int = 1):
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    F, H, W = frames.shape[:3]
    out = np.empty((F * (H // th) * (W // tw), 3 * bins), dtype=np.float32)
    rc = ref().ref_featurize_tiles(_p(frames), F, H, W, th, tw, bins, _p(out), threads)
    if rc:
        raise RuntimeError(f"reference featurize failed: {rc} {ref().ref_last_error()}")
    return out


def ref_color_histogram(px: np.ndarray, bins: int) -> np.ndarray:
    px = np.ascontiguousarray(px, dtype=np.float32)
    n, h, w = px.shape[:3]
    out = np.empty((n, 3 * bins), dtype=np.float32)
    rc = ref().ref_color_histogram_f32(_p(px), n, h, w, bins, _p(out))
    if rc:
        return rc
    return out


def ref_sim_join(L: np.ndarray, R: np.ndarray, tau: float, side: int = 0):
    """sim_join_pairs positions in reference emission order + probe count,
    or an int error code (1 ConfigError, 2 ShapeError, 3 MixedDimension ...)."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    R = np.ascontiguousarray(R, dtype=np.float32)
    n = C.c_int64()
    a = C.POINTER(C.c_int32)()
    b = C.POINTER(C.c_int32)()
    pr = C.c_uint64()
    d = L.shape[1] if L.shape[0] else R.shape[1]
    rc = ref().ref_sim_join(_p(L), L.shape[0], _p(R), R.shape[0], d, float(tau), side,
                            C.byref(n), C.byref(a), C.byref(b), C.byref(pr))
    if rc:
        return rc
    k = n.value
    li = np.ctypeslib.as_array(a, (max(k, 1),))[:k].copy()
    ri = np.ctypeslib.as_array(b, (max(k, 1),))[:k].copy()
    ref().ref_free(C.cast(a, C.c_void_p))
    ref().ref_free(C.cast(b, C.c_void_p))
    return li, ri, pr.value


def ref_euclidean(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return ref().ref_euclidean(_p(a), _p(b), a.shape[0])


def ref_join_probe_timed(L, R, tau, self_join, p0, p1, threads):
    L = np.ascontiguousarray(L, dtype=np.float32)
    R = L if self_join else np.ascontiguousarray(R, dtype=np.float32)
    b = C.c_double()
    p = C.c_double()
    n = ref().ref_join_probe_timed(_p(L), L.shape[0], _p(R), R.shape[0], L.shape[1], float(tau),
                                   int(self_join), p0, p1, threads, C.byref(b), C.byref(p))
    return n, b.value, p.value


def ref_join_probe_pairs(L, R, tau, threads):
    """build_balltree(R) + balltree_within(tau) for every row of L (the
    reference's probe loop, src/query.cpp:516-526, over `threads` threads):
    (left, right, build_s, probe_s), pairs in probe order, ascending ids."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    R = np.ascontiguousarray(R, dtype=np.float32)
    a = C.POINTER(C.c_int32)()
    b = C.POINTER(C.c_int32)()
    bs, ps = C.c_double(), C.c_double()
    n = ref().ref_join_probe_pairs(_p(L), L.shape[0], _p(R), R.shape[0], L.shape[1], float(tau),
                                   int(threads), C.byref(a), C.byref(b), C.byref(bs), C.byref(ps))
    if n < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    li = np.ctypeslib.as_array(a, (max(n, 1),))[:n].copy()
    ri = np.ctypeslib.as_array(b, (max(n, 1),))[:n].copy()
    ref().ref_free(C.cast(a, C.c_void_p))
    ref().ref_free(C.cast(b, C.c_void_p))
    return li, ri, bs.value, ps.value


def ref_dedup(X, tau):
    """PlanNode::dedup through execute() on the reference: (rep_of, n_reps),
    or an int error code."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n = X.shape[0]
    rep_of = np.empty(max(n, 1), dtype=np.int64)
    nr = C.c_int64()
    rc = ref().ref_dedup(_p(X), n, X.shape[1], float(tau), _p(rep_of), C.byref(nr))
    if rc:
        return rc
    return rep_of[:n], nr.value


def ref_dedup_stream(X, tau):
    """dedup_stream on the reference: indices of the kept patches."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    kept = np.empty(max(X.shape[0], 1), dtype=np.int64)
    m = ref().ref_dedup_stream(_p(X), X.shape[0], X.shape[1], float(tau), _p(kept))
    if m < 0:
        return int(-m)
    return kept[:m]


def _ref_pairs(fn, *args):
    n = C.c_int64()
    a = C.POINTER(C.c_int32)()
    b = C.POINTER(C.c_int32)()
    rc = fn(*args, C.byref(n), C.byref(a), C.byref(b))
    if rc:
        return rc
    k = n.value
    x = np.ctypeslib.as_array(a, (max(k, 1),))[:k].copy()
    y = np.ctypeslib.as_array(b, (max(k, 1),))[:k].copy()
    ref().ref_free(C.cast(a, C.c_void_p))
    ref().ref_free(C.cast(b, C.c_void_p))
    return x, y


def ref_nl_within(L, R, radius):
    """PlanNode::nl_join(..., within_of(0, 1, radius)) positions in the
    nested-loop emission order, or an int error code."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    R = np.ascontiguousarray(R, dtype=np.float32)
    d = L.shape[1] if L.shape[0] else R.shape[1]
    return _ref_pairs(ref().ref_nl_within, _p(L), L.shape[0], _p(R), R.shape[0], d, float(radius))


def ref_q1(frames, bins, tau):
    """The reference's q1 plan over whole-frame histograms: (frame a, frame b)
    per result tuple in emission order."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    F, H, W = frames.shape[:3]
    return _ref_pairs(ref().ref_q1, _p(frames), F, H, W, int(bins), float(tau))


def ref_store_write(frames, path, layout=0, quant_step=0, clip_len=64):
    """VideoStore::ingest of frames 0..F-1 (layout 0 frame_file, 1
    encoded_file, 2 segmented_file; quant_step 0 = lossless)."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    F, H, W = frames.shape[:3]
    return ref().ref_store_write(_p(frames), F, H, W, layout, quant_step, clip_len,
                                 str(path).encode())


def ref_store_scan(path, F, H, W, lo=-1, hi=-1):
    """VideoStore::open(path).scan([lo, hi)) decoded frames."""
    n = F if lo < 0 else hi - lo
    out = np.empty((max(n, 1), H, W, 3), np.uint8)
    k = ref().ref_store_scan(str(path).encode(), lo, hi, _p(out))
    if k < 0:
        return int(-k)
    return out[:k]


def ref_run_query(plan, with_data=False, reset_ids=1):
    """patchdb.run_query on the reference (bindings/py_module.cpp:168-213):
    the plan file's ETL section materialized, its plan executed.  Returns
    {"tuples": [[patch, ...], ...]} (patch: id, shape, meta, lineage, data)
    or raises RuntimeError with the reference's message."""
    import json
    if not isinstance(plan, str):
        plan = json.dumps(plan)
    L = ref()
    ptr = L.ref_run_query(plan.encode(), int(bool(with_data)), int(reset_ids))
    if not ptr:
        raise RuntimeError(L.ref_last_error().decode())
    try:
        return json.loads(C.string_at(ptr).decode())
    finally:
        L.ref_free(C.c_void_p(ptr))

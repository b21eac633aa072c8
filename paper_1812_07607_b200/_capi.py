"""ctypes binding of libpdb_cuda.so (include/pdb_cuda.h).

This module is the only place Python touches the C-ABI.  It loads the
in-tree library and fails loudly when it is missing: there is no CPU
fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PDB_CUDA_LIB points at an alternative build (kernel-variant experiments).
LIB_PATH = os.environ.get("PDB_CUDA_LIB") or os.path.join(_HERE, "libpdb_cuda.so")
GEN_PATH = os.path.join(_HERE, "libpdb_gen.so")

PDB_OK = 0
PDB_ERR_CONFIG = 1
PDB_ERR_SHAPE = 2
PDB_ERR_MIXED_DIMENSION = 3
PDB_ERR_DIMENSION_MISMATCH = 4
PDB_ERR_DUPLICATE_ID = 5
PDB_ERR_CAPACITY = 6
PDB_ERR_INVALID_ARGUMENT = 7
PDB_ERR_CUDA = 10
PDB_ERR_OUT_OF_MEMORY = 11
PDB_ERR_NO_DEVICE = 12
PDB_ERR_IO = 13

PDB_HIST_PER_CHANNEL = 0
PDB_HIST_JOINT = 1
PDB_JOIN_SELF = 1
PDB_JOIN_SORTED = 2
PDB_JOIN_TF32 = 4
PDB_JOIN_PHASE_TIMES = 8
PDB_JOIN_DENSE = 16

# Every symbol include/pdb_cuda.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "pdb_last_error", "pdb_status_name", "pdb_version", "pdb_device_count",
    "pdb_hist_dim", "pdb_featurize_tiles", "pdb_featurize_tiles_dev",
    "pdb_color_histogram_f32", "pdb_color_histogram_f32_dev",
    "pdb_sim_join", "pdb_pairs_free", "pdb_sim_join_dev", "pdb_dev_pairs_free",
    "pdb_featurize_join", "pdb_host_alloc", "pdb_host_free",
    "pdb_cosine_join_bf16", "pdb_cosine_join_bf16_dev", "pdb_dedup", "pdb_dedup_dev",
    "pdb_store_open", "pdb_store_close", "pdb_store_describe", "pdb_store_read",
    "pdb_store_featurize", "pdb_rows_within", "pdb_featurize_tiles_dev_multi",
    "pdb_release_caches", "pdb_warmup", "pdb_featurize_join_dev",
)


class StoreInfo(C.Structure):
    _fields_ = [("frame_count", C.c_int64), ("width", C.c_int32), ("height", C.c_int32),
                ("layout", C.c_int32), ("codec_mode", C.c_int32), ("quant_step", C.c_int32),
                ("clip_len", C.c_int32), ("video_id", C.c_char * 256)]


class JoinOpts(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("shard_index", C.c_int32),
                ("shard_count", C.c_int32), ("reserved0", C.c_int32),
                ("stream", C.c_void_p)]


class Pairs(C.Structure):
    _fields_ = [("count", C.c_int64), ("left", C.POINTER(C.c_int32)),
                ("right", C.POINTER(C.c_int32)), ("dist", C.POINTER(C.c_float))]


class DevPairs(C.Structure):
    _fields_ = [("count", C.c_int64), ("capacity", C.c_int64),
                ("left", C.c_void_p), ("right", C.c_void_p), ("dist", C.c_void_p)]


class JoinStats(C.Structure):
    _fields_ = [("candidates", C.c_int64), ("pairs", C.c_int64), ("tiles", C.c_int64),
                ("candidate_capacity", C.c_int64), ("launches", C.c_int32),
                ("screen_passes", C.c_int32), ("prep_ms", C.c_float), ("screen_ms", C.c_float),
                ("recheck_ms", C.c_float), ("sort_ms", C.c_float),
                ("screen_format", C.c_int32), ("reserved1", C.c_int32)]


_lib: Optional[C.CDLL] = None
_gen: Optional[C.CDLL] = None


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(
            f"{os.path.basename(path)} is not built ({path}); run "
            "`python -c 'import __graft_entry__ as g; g.build()'` -- the product "
            "has no CPU fallback")
    return C.CDLL(path)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = _load(LIB_PATH)
        i64, i32, f64, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        L.pdb_last_error.restype = C.c_char_p
        L.pdb_status_name.restype = C.c_char_p
        L.pdb_status_name.argtypes = [C.c_int]
        L.pdb_hist_dim.argtypes = [i32, i32]
        L.pdb_featurize_tiles.argtypes = [vp, i64, i32, i32, i32, i32, i32, i32, vp]
        L.pdb_featurize_tiles_dev.argtypes = [vp, i64, i32, i32, i32, i32, i32, i32, vp, vp]
        L.pdb_color_histogram_f32.argtypes = [vp, i64, i32, i32, i32, i32, vp]
        L.pdb_color_histogram_f32_dev.argtypes = [vp, i64, i32, i32, i32, i32, vp, vp]
        L.pdb_sim_join.argtypes = [vp, i64, vp, i64, i32, f64, C.POINTER(JoinOpts),
                                   C.POINTER(Pairs)]
        L.pdb_pairs_free.argtypes = [C.POINTER(Pairs)]
        L.pdb_pairs_free.restype = None
        L.pdb_sim_join_dev.argtypes = [vp, i64, vp, i64, i32, f64, C.POINTER(JoinOpts),
                                       C.POINTER(DevPairs), C.POINTER(JoinStats)]
        L.pdb_dev_pairs_free.argtypes = [C.POINTER(DevPairs)]
        L.pdb_dev_pairs_free.restype = None
        L.pdb_featurize_join.argtypes = [vp, i64, i32, i32, i32, i32, i32, i32, f64,
                                         C.POINTER(JoinOpts), vp, C.POINTER(Pairs)]
        L.pdb_featurize_join_dev.argtypes = [vp, i64, i32, i32, i32, i32, i32, i32, f64,
                                             C.POINTER(JoinOpts), vp, C.POINTER(DevPairs),
                                             C.POINTER(JoinStats)]
        L.pdb_cosine_join_bf16.argtypes = [vp, i64, vp, i64, i32, f64, C.POINTER(JoinOpts),
                                           C.POINTER(Pairs)]
        L.pdb_cosine_join_bf16_dev.argtypes = [vp, i64, vp, i64, i32, f64, C.POINTER(JoinOpts),
                                               C.POINTER(DevPairs), C.POINTER(JoinStats)]
        L.pdb_dedup.argtypes = [vp, i64, i32, f64, C.POINTER(JoinOpts), vp, C.POINTER(i64)]
        L.pdb_dedup_dev.argtypes = [vp, i64, i32, f64, C.POINTER(JoinOpts), vp, C.POINTER(i64)]
        L.pdb_store_open.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.pdb_store_close.argtypes = [vp]
        L.pdb_store_close.restype = None
        L.pdb_store_describe.argtypes = [vp, C.POINTER(StoreInfo)]
        L.pdb_store_read.argtypes = [vp, i64, i64, vp, C.POINTER(i64), i32]
        L.pdb_store_featurize.argtypes = [vp, i64, i64, i32, i32, i32, i32, vp, C.POINTER(i64),
                                          i32, vp]
        L.pdb_rows_within.argtypes = [vp, vp, i64, i32, f64, vp]
        L.pdb_featurize_tiles_dev_multi.argtypes = [vp, i64, i32, i32, i32, i32, i32, i32, vp, i32,
                                                    vp]
        L.pdb_release_caches.argtypes = []
        L.pdb_warmup.argtypes = []
        L.pdb_host_alloc.argtypes = [i64]
        L.pdb_host_alloc.restype = vp
        L.pdb_host_free.argtypes = [vp]
        L.pdb_host_free.restype = None
        _lib = L
    return _lib


def gen() -> C.CDLL:
    global _gen
    if _gen is None:
        G = _load(GEN_PATH)
        i64, i32, f64, u64, vp = C.c_int64, C.c_int32, C.c_double, C.c_uint64, C.c_void_p
        G.pdb_gen_clusters.argtypes = [vp, i64, i32, i32, f64, i32, u64, u64, i32]
        G.pdb_gen_plant.argtypes = [vp, i64, vp, i64, i32, f64, f64, u64, vp, vp, i64]
        G.pdb_gen_plant.restype = i64
        G.pdb_gen_simplex.argtypes = [vp, i64, i32, i32, f64, f64, u64, i32]
        G.pdb_gen_uniform.argtypes = [vp, i64, i32, u64, i32]
        G.pdb_gen_frames.argtypes = [vp, i64, i64, i32, i32, i32, i32, i32, i32, u64, vp, i32]
        _gen = G
    return _gen


def ptr(a) -> int:
    """Address of a numpy array or torch tensor (contiguous)."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def last_error() -> str:
    return lib().pdb_last_error().decode()


def status_name(st: int) -> str:
    return lib().pdb_status_name(st).decode()

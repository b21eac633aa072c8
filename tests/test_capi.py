"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/pdb_cuda.h declares, validates arguments with the reference's error
taxonomy, and -- with no sm_100 device -- refuses to compute (no CPU path)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1812_07607_b200 import _capi as capi
from paper_1812_07607_b200 import patchdb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "pdb_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(pdb_[a-z0-9_]+)\s*\(", src))


def test_exports_every_declared_symbol():
    lib = capi.lib()
    declared = _header_symbols()
    assert declared == set(capi.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_exports_nothing_else():
    out = os.popen(f"nm -D --defined-only {capi.LIB_PATH}").read()
    syms = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert {s for s in syms if s.startswith("pdb_")} == set(capi.EXPORTS)


def test_hist_dim():
    lib = capi.lib()
    assert lib.pdb_hist_dim(4, 0) == 12
    assert lib.pdb_hist_dim(8, 0) == 24
    assert lib.pdb_hist_dim(4, 1) == 64
    assert lib.pdb_hist_dim(16, 1) == 4096
    assert lib.pdb_hist_dim(17, 1) == -1
    assert lib.pdb_hist_dim(1, 0) == -1


def test_validation_errors_before_device():
    lib = capi.lib()
    fr = np.zeros((1, 8, 8, 3), np.uint8)
    out = np.zeros((1, 64), np.float32)
    # bins < 2 -> ConfigError (src/etl.cpp:64-67)
    assert lib.pdb_featurize_tiles(capi.ptr(fr), 1, 8, 8, 8, 8, 1, 0, capi.ptr(out)) == capi.PDB_ERR_CONFIG
    assert "bins" in capi.last_error()
    # tile < 1 -> ConfigError (src/etl.cpp:47-50)
    assert lib.pdb_featurize_tiles(capi.ptr(fr), 1, 8, 8, 0, 8, 4, 0, capi.ptr(out)) == capi.PDB_ERR_CONFIG
    # joint with B > 16 -> ConfigError
    assert lib.pdb_featurize_tiles(capi.ptr(fr), 1, 8, 8, 8, 8, 17, 1, capi.ptr(out)) == capi.PDB_ERR_CONFIG
    # bad mode
    assert lib.pdb_featurize_tiles(capi.ptr(fr), 1, 8, 8, 8, 8, 4, 7, capi.ptr(out)) == capi.PDB_ERR_INVALID_ARGUMENT
    # non-pixel float patches -> ShapeError (src/etl.cpp:332-334)
    px = np.zeros((1, 4, 4, 3), np.float32)
    assert lib.pdb_color_histogram_f32(capi.ptr(px), 1, 0, 4, 4, 0, capi.ptr(out)) == capi.PDB_ERR_SHAPE
    # tau < 0 -> ConfigError (src/query.cpp:488)
    L = np.zeros((3, 2), np.float32)
    pr = capi.Pairs()
    assert lib.pdb_sim_join(capi.ptr(L), 3, capi.ptr(L), 3, 2, -1.0, None, C.byref(pr)) == capi.PDB_ERR_CONFIG
    # NaN tau passes validation like the reference's `tau < 0.0` check (it then
    # needs the device: no CPU path), so it is no ConfigError
    assert lib.pdb_sim_join(capi.ptr(L), 3, capi.ptr(L), 3, 2, float("nan"), None, C.byref(pr)) != capi.PDB_ERR_CONFIG
    # d == 0 with rows -> ShapeError (src/query.cpp:467-477)
    assert lib.pdb_sim_join(capi.ptr(L), 3, capi.ptr(L), 3, 0, 1.0, None, C.byref(pr)) == capi.PDB_ERR_SHAPE
    o = capi.JoinOpts()
    o.flags = 1 << 7
    assert lib.pdb_sim_join(capi.ptr(L), 3, capi.ptr(L), 3, 2, 1.0, C.byref(o), C.byref(pr)) == capi.PDB_ERR_INVALID_ARGUMENT


def test_object_api_errors_mirror_reference():
    with pytest.raises(patchdb.ConfigError):
        patchdb.sim_join_pairs([], [], -0.1)
    a = patchdb.Patch(1, np.zeros(3, np.float32), (3,))
    b = patchdb.Patch(2, np.zeros(2, np.float32), (2,))
    with pytest.raises(patchdb.MixedDimensionError):
        patchdb.sim_join_pairs([a, b], [a], 0.5)
    with pytest.raises(patchdb.DimensionMismatchError):
        patchdb.sim_join_pairs([a], [b], 0.5)
    e = patchdb.Patch(3, np.zeros(0, np.float32), (0,))
    with pytest.raises(patchdb.ShapeError):
        patchdb.sim_join_pairs([e], [a], 0.5)
    # empty sides -> no pairs, no device needed
    assert patchdb.sim_join_pairs([], [a], 0.5) == []
    assert patchdb.sim_join_pairs([a], [], 0.5) == []
    # duplicate ids on the build side (src/query.cpp:508-514)
    a2 = patchdb.Patch(1, np.ones(3, np.float32), (3,))
    with pytest.raises(patchdb.DuplicatePatchIdError):
        patchdb.sim_join_pairs([a, a2], [a, a2, a], 0.5)
    with pytest.raises(patchdb.ConfigError):
        patchdb.TransformerSpec(bins=1).validate()
    with pytest.raises(patchdb.ShapeError):
        patchdb.apply_transformer(a, patchdb.TransformerSpec(bins=4))
    with pytest.raises(patchdb.ConfigError):
        patchdb.GeneratorSpec("tiles", 0, 3).validate()


def test_generate_tiles_grid_and_lineage():
    # test_etl.cpp:91-115: 14x8 frame, 4x3 tiles -> 3x2 grid, partial edges dropped
    fr = patchdb.Frame("v", 0, np.zeros((8, 14, 3), np.uint8))
    patchdb.reset_patch_ids()
    out = list(patchdb.generate([fr], patchdb.GeneratorSpec("tiles", 4, 3)))
    assert len(out) == 6
    assert [p.meta["bbox"][:2] for p in out] == [(0, 0), (4, 0), (8, 0), (0, 3), (4, 3), (8, 3)]
    assert all(p.shape == (3, 4, 3) for p in out)
    assert [p.patch_id for p in out] == [1, 2, 3, 4, 5, 6]
    assert out[0].lineage[0].op_name == "make_patch"


@pytest.mark.skipif(capi.lib().pdb_device_count() > 0, reason="a GPU is present")
def test_no_cpu_fallback_without_device():
    lib = capi.lib()
    fr = np.zeros((1, 8, 8, 3), np.uint8)
    out = np.zeros((1, 12), np.float32)
    assert lib.pdb_featurize_tiles(capi.ptr(fr), 1, 8, 8, 8, 8, 4, 0, capi.ptr(out)) == capi.PDB_ERR_NO_DEVICE
    L = np.zeros((3, 2), np.float32)
    pr = capi.Pairs()
    assert lib.pdb_sim_join(capi.ptr(L), 3, capi.ptr(L), 3, 2, 1.0, None, C.byref(pr)) == capi.PDB_ERR_NO_DEVICE
    with pytest.raises(patchdb.DeviceError):
        patchdb.featurize_tiles(fr, 8, 8, 4)

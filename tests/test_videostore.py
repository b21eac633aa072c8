"""Frame source: libpdb_cuda's reader of the reference's
VideoStore files against the reference's own scan of the same files
(tests/golden/stores, written by VideoStore::ingest; make_golden.py stores).
Decoding is host work (zlib), so these run without a GPU."""

import hashlib
import os

import numpy as np
import pytest

from paper_1812_07607_b200 import patchdb

SDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "stores")
NAMES = ["frame_file", "encoded_lossless", "encoded_lossy16", "segmented_lossless_c5",
         "segmented_lossy4_c8"]


def _gold():
    return np.load(os.path.join(SDIR, "stores_golden.npz"))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()


@pytest.mark.parametrize("name", NAMES)
def test_scan_matches_reference_decode(name):
    z = _gold()
    st = patchdb.VideoStore.open(os.path.join(SDIR, f"{name}.pdb"))
    assert (st.frame_count, st.height, st.width) == (16, 32, 48)
    full = st.scan_array()
    assert _sha(full) == z[f"{name}__full_sha"].tobytes()
    part = st.scan_array((3, 13))
    assert part.shape[0] == 10 and _sha(part) == z[f"{name}__part_sha"].tobytes()
    frames = list(st.scan((3, 13)))
    assert [f.frame_no for f in frames] == list(range(3, 13))
    assert np.array_equal(np.stack([f.pixels for f in frames]), part)


def test_scan_range_rules_and_errors(tmp_path):
    st = patchdb.VideoStore.open(os.path.join(SDIR, "segmented_lossless_c5.pdb"))
    with pytest.raises(patchdb.ConfigError):
        st.scan_array((5, 5))
    assert st.scan_array((14, 100)).shape[0] == 2      # clamped to the frame count
    assert st.scan_array((20, 30)).shape[0] == 0
    bad = tmp_path / "bad.pdb"
    bad.write_bytes(b"PDBS0001" + b"\0" * 40)
    with pytest.raises(patchdb.IoError):
        patchdb.VideoStore.open(str(bad))
    with pytest.raises(patchdb.IoError):
        patchdb.VideoStore.open(str(tmp_path / "missing.pdb"))


def test_lossless_round_trip_of_generator_frames():
    from paper_1812_07607_b200 import workloads
    fr, _ = workloads.frames(16, 32, 48, seed=7, block=8, noise=2, period=6)
    z = _gold()
    for name in NAMES:
        if int(z[f"{name}__lossless"][0]):
            got = patchdb.VideoStore.open(os.path.join(SDIR, f"{name}.pdb")).scan_array()
            assert np.array_equal(got, fr), name

"""K1 parity on the B200: bit-exact against the reference's golden outputs
and the C restatement, through the C-ABI (host and device entry points)."""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_1812_07607_b200 import patchdb, workloads
from tests import golden_io

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_golden_per_channel_host_entry():
    for name, fr, th, tw, b, want in golden_io.hist_cases():
        got = patchdb.featurize_tiles(fr, th, tw, b, "per_channel")
        assert np.array_equal(_bits(got), _bits(want)), name


def test_golden_per_channel_device_entry():
    for name, fr, th, tw, b, want in golden_io.hist_cases():
        dev = torch.from_numpy(np.ascontiguousarray(fr)).cuda()
        got = patchdb.featurize_tiles(dev, th, tw, b, "per_channel").cpu().numpy()
        assert np.array_equal(_bits(got), _bits(want)), name


@pytest.mark.parametrize("bins", [2, 3, 4, 5, 8, 16])
def test_joint_matches_restated_oracle(bins):
    fr, _ = workloads.frames(6, 480, 640, seed=11)
    got = patchdb.featurize_tiles(fr, 60, 80, bins, "joint")
    want = oracle.featurize_tiles(fr, 60, 80, bins, 1)
    assert np.array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("shape", [(37, 53, 7, 9), (64, 96, 16, 32), (480, 640, 480, 640),
                                   (50, 80, 25, 16), (48, 64, 12, 16)])
@pytest.mark.parametrize("bins,mode", [(4, 0), (8, 0), (21, 0), (22, 0), (300, 0), (4, 1), (7, 1)])
def test_shapes_and_bins(shape, bins, mode):
    H, W, th, tw = shape
    rng = np.random.default_rng(H * 7 + W + bins)
    fr = rng.integers(0, 256, (3, H, W, 3), dtype=np.uint8)
    got = patchdb.featurize_tiles(fr, th, tw, bins, mode)
    want = oracle.featurize_tiles(fr, th, tw, bins, mode)
    assert np.array_equal(_bits(got), _bits(want))


def test_config2_full_size_properties():
    """Full config-2 frame count: per-channel marginals of the joint
    histogram equal the per-channel histogram, L1 mass 1, and a sampled
    set of frames is bit-exact against the oracle."""
    fr, src = workloads.frames(1000, 480, 640, seed=2)
    dev = torch.from_numpy(fr).cuda()
    j = patchdb.featurize_tiles(dev, 60, 80, 4, "joint")
    p = patchdb.featurize_tiles(dev, 60, 80, 4, "per_channel")
    assert j.shape == (64000, 64) and p.shape == (64000, 12)
    cnt = torch.round(j.double() * 4800).long().view(-1, 4, 4, 4)
    pc = torch.round(p.double() * 4800).long().view(-1, 3, 4)
    assert torch.equal(cnt.sum((2, 3)), pc[:, 0])
    assert torch.equal(cnt.sum((1, 3)), pc[:, 1])
    assert torch.equal(cnt.sum((1, 2)), pc[:, 2])
    assert torch.equal(cnt.sum((1, 2, 3)), torch.full((64000,), 4800, device="cuda"))
    jh = j.cpu().numpy()
    for f in (0, 19, 500, 999):
        want = oracle.featurize_tiles(fr[f:f + 1], 60, 80, 4, 1)
        assert np.array_equal(_bits(jh[f * 64:(f + 1) * 64]), _bits(want))


def test_f32_patch_path_golden_and_clamp():
    px, want = golden_io.f32_case()
    got = patchdb.color_histogram(px, 8, "per_channel")
    assert np.array_equal(_bits(got), _bits(want))
    # joint over the same float patches vs the restatement
    assert np.array_equal(_bits(patchdb.color_histogram(px, 4, "joint")),
                          _bits(oracle.color_histogram(px, 4, 1)))
    # large per-channel D takes the global-counter path
    rng = np.random.default_rng(3)
    px2 = rng.integers(0, 256, (3, 20, 20, 3)).astype(np.float32)
    assert np.array_equal(_bits(patchdb.color_histogram(px2, 5000, 0)),
                          _bits(oracle.color_histogram(px2, 5000, 0)))


def test_object_api_transform_matches_reference_shape_and_lineage():
    fr = workloads.frames(2, 48, 64, seed=4)[0]
    frames = [patchdb.Frame("v", i, fr[i]) for i in range(2)]
    patchdb.reset_patch_ids()
    pix = list(patchdb.generate(frames, patchdb.GeneratorSpec("tiles", 16, 12)))
    out = list(patchdb.transform(pix, patchdb.TransformerSpec(bins=4)))
    assert len(out) == 2 * 4 * 4
    assert all(p.shape == (12,) and len(p.lineage) == 2 for p in out)
    want = oracle.featurize_tiles(fr, 12, 16, 4, 0)
    assert np.array_equal(_bits(np.stack([p.data for p in out])), _bits(want))


def test_empty_and_degenerate():
    fr = np.zeros((0, 8, 8, 3), np.uint8)
    assert patchdb.featurize_tiles(fr, 4, 4, 4).shape[0] == 0
    fr = np.zeros((2, 8, 8, 3), np.uint8)
    assert patchdb.featurize_tiles(fr, 9, 4, 4).shape[0] == 0   # tile taller than the frame


@pytest.mark.parametrize("H,W,th,tw", [
    (90, 640, 90, 80),     # 15 batches of 6 rows: 240 pixels per lane (8-bit counter limit)
    (91, 640, 91, 80),     # 16 batches -> over the 8-bit limit, LDG-staged fallback
    (120, 256, 60, 16),    # 16 tile columns, 48-byte tile rows
    (120, 272, 60, 16),    # 17 tile columns -> fallback
    (70, 160, 35, 80),     # partial last batch (35 = 5*6 + 5)
    (96, 192, 32, 64),     # 192-byte tile rows
    (64, 96, 64, 32),
])
@pytest.mark.parametrize("bins", [2, 4])
@pytest.mark.parametrize("content", ["uniform", "solid", "blocks"])
def test_joint_tma_kernel_edges(H, W, th, tw, bins, content):
    """The TMA-fed 8-bit-counter kernel (and its fallbacks) at its shape
    limits; solid frames put every pixel of a lane in one counter."""
    rng = np.random.default_rng(H + W + th + tw + bins)
    if content == "uniform":
        fr = rng.integers(0, 256, (5, H, W, 3), dtype=np.uint8)
    elif content == "solid":
        fr = np.empty((5, H, W, 3), np.uint8)
        fr[:] = rng.integers(0, 256, (5, 1, 1, 3), dtype=np.uint8)
    else:
        fr, _ = workloads.frames(5, H, W, seed=H + W)
    dev = torch.from_numpy(fr).cuda()
    got = patchdb.featurize_tiles(dev, th, tw, bins, "joint").cpu().numpy()
    want = oracle.featurize_tiles(fr, th, tw, bins, 1)
    assert np.array_equal(_bits(got), _bits(want))


def test_joint_tma_kernel_offset_frames():
    """Frames starting at a 16-byte but not 128-byte aligned device address,
    and a frame count that leaves CTAs with unequal tile-row counts."""
    fr, _ = workloads.frames(37, 480, 640, seed=5)
    big = torch.empty(fr.nbytes + 64, dtype=torch.uint8, device="cuda")
    view = big[16:16 + fr.nbytes].view(37, 480, 640, 3)
    view.copy_(torch.from_numpy(fr))
    got = patchdb.featurize_tiles(view, 60, 80, 4, "joint").cpu().numpy()
    want = oracle.featurize_tiles(fr, 60, 80, 4, 1)
    assert np.array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("name", ["frame_file", "encoded_lossy16", "segmented_lossy4_c8"])
def test_store_featurize_matches_featurizing_the_decoded_frames(name):
    """pdb_store_featurize (decode chunk by chunk + K1) equals K1 on the
    frames the reference's scan decodes, and the restatement on them."""
    import os
    sdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "stores")
    st = patchdb.VideoStore.open(os.path.join(sdir, f"{name}.pdb"))
    fr = st.scan_array()
    for bins, mode, th, tw in [(4, "joint", 8, 16), (8, "per_channel", 16, 16), (2, "joint", 32, 48)]:
        got = st.featurize(th, tw, bins, mode).cpu().numpy()
        want = oracle.featurize_tiles(fr, th, tw, bins, 1 if mode == "joint" else 0)
        assert np.array_equal(_bits(got), _bits(want)), (name, bins, mode)
        part = st.featurize(th, tw, bins, mode, rng=(3, 13)).cpu().numpy()
        want_p = oracle.featurize_tiles(fr[3:13], th, tw, bins, 1 if mode == "joint" else 0)
        assert np.array_equal(_bits(part), _bits(want_p))


@pytest.mark.parametrize("shape", [(60, 80, 4, 1), (16, 16, 4, 1), (60, 80, 8, 0)])
def test_featurize_multi_output_writes_every_buffer(shape):
    """pdb_featurize_tiles_dev_multi (the fused feature all-gather): every
    output buffer holds the single-output features, at the given offset --
    the TMA kernel's multi-output stores (60x80 joint B=4) and the
    copy-to-peers fallback (other shapes)."""
    import ctypes as C
    import torch
    from paper_1812_07607_b200 import _capi as capi
    th, tw, bins, mode = shape
    fr, _ = workloads.frames(12, 480, 640, seed=9)
    d_fr = torch.from_numpy(fr).cuda()
    D = capi.lib().pdb_hist_dim(bins, mode)
    n = 12 * (480 // th) * (640 // tw)
    want = patchdb.featurize_tiles(fr, th, tw, bins, "joint" if mode else "per_channel")
    bufs = [torch.full((n + 7, D), -1.0, device="cuda") for _ in range(3)]
    ptrs = (C.c_void_p * 3)(*[b.data_ptr() + 7 * D * 4 for b in bufs])
    s = torch.cuda.current_stream()
    rc = capi.lib().pdb_featurize_tiles_dev_multi(d_fr.data_ptr(), 12, 480, 640, th, tw, bins, mode,
                                                  ptrs, 3, C.c_void_p(s.cuda_stream))
    assert rc == 0, capi.last_error()
    torch.cuda.synchronize()
    for b in bufs:
        got = b[7:].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.reshape(n, D).view(np.uint32))
        assert (b[:7].cpu().numpy() == -1.0).all()

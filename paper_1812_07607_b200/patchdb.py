"""Host-side mirror of the reference ``patchdb`` operator interface for the
hot path, running on the B200 kernels behind include/pdb_cuda.h.

Mirrors (paths relative to the reference's proj/ directory):

* errors                     include/patchdb/core.hpp:22-47  (Python sees
                             RuntimeError subclasses, as tests/python expects)
* Frame, Patch               include/patchdb/core.hpp:66-141
* GeneratorSpec, TransformerSpec, generate, transform, apply_transformer
                             include/patchdb/etl.hpp:32-74, src/etl.cpp:252-373
* BuildSide, sim_join_pairs  include/patchdb/query.hpp:84, 206-211,
                             src/query.cpp:467-528, 1094-1104
* nl_join_within            PlanNode::nl_join with a within predicate,
                             include/patchdb/query.hpp:135, src/query.cpp:142-151, 705-744
* q1_duplicate_frames        the q1 near-duplicate-frame plan, src/bench.cpp:695-730
* VideoStore (open, scan, featurize)  the frame source: the reference's
                             store files, include/patchdb/storage.hpp:60-89,
                             src/storage.cpp:170-501, src/record_store.cpp
* dedup_groups, dedup_stream PlanNode::dedup / dedup_stream,
                             include/patchdb/query.hpp:142, 203-204,
                             src/query.cpp:535-582, 1063-1092

Array entry points (featurize_tiles, color_histogram, sim_join,
sim_join_device, featurize_join) are the C-ABI one level down; the object
API above them reproduces the reference's argument checks, error types,
output shapes and emission order.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, Iterator, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as capi

# ---------------------------------------------------------------------------
# Errors (core.hpp:22-47)


class Error(RuntimeError):
    """patchdb::Error"""


class ConfigError(Error):
    pass


class ShapeError(Error):
    pass


class MixedDimensionError(Error):
    pass


class DimensionMismatchError(Error):
    pass


class DuplicatePatchIdError(Error):
    pass


class RegionOutOfBoundsError(Error):
    pass


class IoError(Error):
    """patchdb::IoError (unreadable / malformed store file)."""


class ValidationError(Error):
    """patchdb::ValidationError (plan files, pipeline checks, tuple widths)."""


class TagMismatchError(Error):
    pass


class MissingKeyError(Error):
    pass


class MalformedLineageError(Error):
    pass


class DeviceError(Error):
    """CUDA failure, missing sm_100 device or out-of-memory (no CPU path)."""


_STATUS_EXC = {
    capi.PDB_ERR_CONFIG: ConfigError,
    capi.PDB_ERR_SHAPE: ShapeError,
    capi.PDB_ERR_MIXED_DIMENSION: MixedDimensionError,
    capi.PDB_ERR_DIMENSION_MISMATCH: DimensionMismatchError,
    capi.PDB_ERR_DUPLICATE_ID: DuplicatePatchIdError,
    capi.PDB_ERR_IO: IoError,
}


def _check(status: int) -> None:
    if status == capi.PDB_OK:
        return
    exc = _STATUS_EXC.get(status)
    msg = capi.last_error()
    if exc is not None:
        raise exc(msg)
    if status == capi.PDB_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise DeviceError(f"{capi.status_name(status)}: {msg}")


# ---------------------------------------------------------------------------
# Array-level operators (one C-ABI call each)

HIST_MODES = {"per_channel": capi.PDB_HIST_PER_CHANNEL, "joint": capi.PDB_HIST_JOINT}


def _mode(mode) -> int:
    return HIST_MODES[mode] if isinstance(mode, str) else int(mode)


def hist_dim(bins: int, mode="per_channel") -> int:
    return capi.lib().pdb_hist_dim(bins, _mode(mode))


def featurize_tiles(frames, tile_h: int, tile_w: int, bins: int = 8, mode="per_channel",
                    stream=None):
    """generate(tiles) -> transform(color_histogram) fused (K1).

    ``frames``: uint8 [F, H, W, 3].  A numpy array runs the host entry point
    (copy in, K1, copy out) and returns numpy; a CUDA torch tensor runs the
    device entry point on ``stream`` and returns a CUDA tensor.
    Output [F * (H // tile_h) * (W // tile_w), D], tiles in reference emission
    order (src/etl.cpp:264-298).
    """
    m = _mode(mode)
    F, H, W = (int(frames.shape[0]), int(frames.shape[1]), int(frames.shape[2]))
    if frames.ndim != 4 or frames.shape[3] != 3:
        raise ShapeError("frames must be [F, H, W, 3] uint8")
    if bins >= 2 and tile_h >= 1 and tile_w >= 1:
        D = hist_dim(bins, m)
        n = F * (H // tile_h) * (W // tile_w)
    else:
        D, n = 1, 0
    if isinstance(frames, np.ndarray):
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        out = np.empty((n, max(D, 1)), dtype=np.float32)
        _check(capi.lib().pdb_featurize_tiles(capi.ptr(frames), F, H, W, tile_h, tile_w, bins,
                                              m, capi.ptr(out)))
        return out
    import torch
    assert frames.is_cuda and frames.dtype == torch.uint8 and frames.is_contiguous()
    out = torch.empty((n, max(D, 1)), dtype=torch.float32, device=frames.device)
    s = stream if stream is not None else torch.cuda.current_stream(frames.device)
    _check(capi.lib().pdb_featurize_tiles_dev(frames.data_ptr(), F, H, W, tile_h, tile_w, bins,
                                              m, out.data_ptr(), C.c_void_p(s.cuda_stream)))
    return out


def color_histogram(patches: np.ndarray, bins: int = 8, mode="per_channel") -> np.ndarray:
    """apply_transformer(color_histogram) over float pixel patches [n, h, w, 3]."""
    m = _mode(mode)
    patches = np.ascontiguousarray(patches, dtype=np.float32)
    if patches.ndim != 4 or patches.shape[3] != 3:
        raise ShapeError("transformer input must be pixel shaped [h,w,3]")
    n, h, w = patches.shape[:3]
    D = hist_dim(bins, m) if bins >= 2 else 1
    out = np.empty((n, max(D, 1)), dtype=np.float32)
    _check(capi.lib().pdb_color_histogram_f32(capi.ptr(patches), n, h, w, bins, m,
                                              capi.ptr(out)))
    return out


@dataclass
class JoinResult:
    left: np.ndarray   # int32 row indices into L
    right: np.ndarray  # int32 row indices into R (into L for self-joins)
    dist: np.ndarray   # float32, the reference's fp64 euclidean rounded to fp32

    def __len__(self) -> int:
        return int(self.left.shape[0])


def _opts(self_join: bool, sort: bool, shard: Tuple[int, int], stream=None,
          tf32: bool = False, phase_times: bool = False, dense: bool = False) -> capi.JoinOpts:
    o = capi.JoinOpts()
    o.flags = ((capi.PDB_JOIN_SELF if self_join else 0) | (capi.PDB_JOIN_SORTED if sort else 0) |
               (capi.PDB_JOIN_TF32 if tf32 else 0) |
               (capi.PDB_JOIN_PHASE_TIMES if phase_times else 0) |
               (capi.PDB_JOIN_DENSE if dense else 0))
    o.shard_index, o.shard_count = int(shard[0]), int(shard[1])
    o.stream = stream
    return o


def sim_join(L: np.ndarray, R: Optional[np.ndarray], tau: float, *, self_join: bool = False,
             sort: bool = True, shard: Tuple[int, int] = (0, 1), tf32: bool = False,
             dense: bool = False) -> JoinResult:
    """Host threshold join (K2 + K3): every (i, j) with euclidean(L_i, R_j) <= tau.

    ``self_join=True`` joins L with itself and keeps i < j.  ``tf32`` screens
    on tf32 instead of bf16 copies (same result, tighter candidate band).
    ``dense`` screens every tile (no band plan; same result).
    """
    L = np.ascontiguousarray(L, dtype=np.float32)
    if L.ndim != 2:
        raise ShapeError("L must be [n, d]")
    if self_join:
        R_, nR = L, L.shape[0]
    else:
        R_ = np.ascontiguousarray(R, dtype=np.float32)
        if R_.ndim != 2:
            raise ShapeError("R must be [n, d]")
        nR = R_.shape[0]
        if L.shape[0] and nR and L.shape[1] != R_.shape[1]:
            raise DimensionMismatchError(
                f"similarity join over {L.shape[1]} and {R_.shape[1]} dimensional sides")
    d = L.shape[1] if L.shape[0] else (R_.shape[1] if nR else L.shape[1])
    o = _opts(self_join, sort, shard, tf32=tf32, dense=dense)
    pr = capi.Pairs()
    _check(capi.lib().pdb_sim_join(capi.ptr(L), L.shape[0], capi.ptr(R_), nR, d, float(tau),
                                   C.byref(o), C.byref(pr)))
    try:
        n = int(pr.count)
        if n:
            left = np.ctypeslib.as_array(pr.left, shape=(n,)).copy()
            right = np.ctypeslib.as_array(pr.right, shape=(n,)).copy()
            dist = np.ctypeslib.as_array(pr.dist, shape=(n,)).copy()
        else:
            left = np.empty(0, np.int32)
            right = np.empty(0, np.int32)
            dist = np.empty(0, np.float32)
    finally:
        capi.lib().pdb_pairs_free(C.byref(pr))
    return JoinResult(left, right, dist)


def _pairs_to_result(pr) -> JoinResult:
    try:
        n = int(pr.count)
        if n:
            return JoinResult(np.ctypeslib.as_array(pr.left, shape=(n,)).copy(),
                              np.ctypeslib.as_array(pr.right, shape=(n,)).copy(),
                              np.ctypeslib.as_array(pr.dist, shape=(n,)).copy())
        return JoinResult(np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.float32))
    finally:
        capi.lib().pdb_pairs_free(C.byref(pr))


def cosine_join_bf16(L: np.ndarray, R: Optional[np.ndarray], min_cos: float, *,
                     self_join: bool = False, sort: bool = True,
                     shard: Tuple[int, int] = (0, 1)) -> JoinResult:
    """Cosine threshold join over bf16 rows given as uint16 bit patterns
    [n, d] (BASELINE config 4, restated).  ``dist`` = fp32(cos)."""
    L = np.ascontiguousarray(L, dtype=np.uint16)
    R_ = L if self_join else np.ascontiguousarray(R, dtype=np.uint16)
    if L.ndim != 2 or R_.ndim != 2:
        raise ShapeError("L and R must be [n, d] uint16 (bf16 bits)")
    if not self_join and L.shape[0] and R_.shape[0] and L.shape[1] != R_.shape[1]:
        raise DimensionMismatchError(
            f"cosine join over {L.shape[1]} and {R_.shape[1]} dimensional sides")
    o = _opts(self_join, sort, shard)
    pr = capi.Pairs()
    _check(capi.lib().pdb_cosine_join_bf16(capi.ptr(L), L.shape[0], capi.ptr(R_), R_.shape[0],
                                           L.shape[1], float(min_cos), C.byref(o), C.byref(pr)))
    return _pairs_to_result(pr)


class DevicePairs:
    """Device-resident join output, reusable across calls (pdb_dev_pairs)."""

    def __init__(self):
        self._p = capi.DevPairs()
        self.stats = capi.JoinStats()

    @property
    def count(self) -> int:
        return int(self._p.count)

    def to_torch(self, device, copy: bool = True):
        """The three arrays (count elements) as CUDA tensors: views of the
        library's device buffers (copy=False) or clones."""
        import torch
        n = self.count
        out = []
        for p_, ts in ((self._p.left, "<i4"), (self._p.right, "<i4"), (self._p.dist, "<f4")):
            if n == 0:
                out.append(torch.empty(0, dtype=torch.float32 if ts == "<f4" else torch.int32,
                                       device=device))
                continue
            v = torch.as_tensor(_CudaArray(p_, n, ts), device=device)
            out.append(v.clone() if copy else v)
        return tuple(out)

    def free(self):
        capi.lib().pdb_dev_pairs_free(C.byref(self._p))

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer."""

    def __init__(self, ptr_: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr_), False), "version": 3,
                                         "strides": None}


def cosine_join_bf16_device(L, R, min_cos: float, *, self_join: bool = False, sort: bool = False,
                            shard: Tuple[int, int] = (0, 1), out: Optional["DevicePairs"] = None,
                            stream=None, phase_times: bool = False) -> "DevicePairs":
    """Device cosine join on CUDA bf16 torch tensors; the result stays in HBM."""
    import torch
    assert L.is_cuda and L.dtype == torch.bfloat16 and L.is_contiguous()
    nL, d = int(L.shape[0]), int(L.shape[1])
    if self_join or R is None:
        Rp, nR = L.data_ptr(), nL
    else:
        assert R.is_cuda and R.dtype == torch.bfloat16 and R.is_contiguous()
        Rp, nR = R.data_ptr(), int(R.shape[0])
    s = stream if stream is not None else torch.cuda.current_stream(L.device)
    o = _opts(self_join, sort, shard, C.c_void_p(s.cuda_stream), phase_times=phase_times)
    res = out if out is not None else DevicePairs()
    _check(capi.lib().pdb_cosine_join_bf16_dev(L.data_ptr(), nL, Rp, nR, d, float(min_cos),
                                               C.byref(o), C.byref(res._p), C.byref(res.stats)))
    return res


def sim_join_device(L, R, tau: float, *, self_join: bool = False, sort: bool = False,
                    shard: Tuple[int, int] = (0, 1), out: Optional[DevicePairs] = None,
                    stream=None, tf32: bool = False, phase_times: bool = False,
                    dense: bool = False) -> DevicePairs:
    """Device threshold join on CUDA torch tensors; the result stays in HBM.
    ``phase_times`` fills ``stats.*_ms`` (CUDA events between the phases);
    ``dense`` screens every tile (no band plan)."""
    import torch
    assert L.is_cuda and L.dtype == torch.float32 and L.is_contiguous()
    nL, d = int(L.shape[0]), int(L.shape[1])
    if self_join or R is None:
        Rp, nR = L.data_ptr(), nL
    else:
        assert R.is_cuda and R.dtype == torch.float32 and R.is_contiguous()
        Rp, nR = R.data_ptr(), int(R.shape[0])
    s = stream if stream is not None else torch.cuda.current_stream(L.device)
    o = _opts(self_join, sort, shard, C.c_void_p(s.cuda_stream), tf32=tf32,
              phase_times=phase_times, dense=dense)
    res = out if out is not None else DevicePairs()
    _check(capi.lib().pdb_sim_join_dev(L.data_ptr(), nL, Rp, nR, d, float(tau), C.byref(o),
                                       C.byref(res._p), C.byref(res.stats)))
    return res


def featurize_join(frames: np.ndarray, tile_h: int, tile_w: int, bins: int, mode, tau: float,
                   *, want_features: bool = False, shard: Tuple[int, int] = (0, 1)):
    """Host frames -> tile histograms -> self-join (i < j) -> host pairs."""
    m = _mode(mode)
    frames = np.ascontiguousarray(frames, dtype=np.uint8) if isinstance(frames, np.ndarray) else frames
    F, H, W = frames.shape[:3]
    D = hist_dim(bins, m)
    feats = None
    fptr = None
    if want_features:
        feats = np.empty((F * (H // tile_h) * (W // tile_w), D), dtype=np.float32)
        fptr = capi.ptr(feats)
    o = _opts(True, True, shard)
    pr = capi.Pairs()
    _check(capi.lib().pdb_featurize_join(capi.ptr(frames), F, H, W, tile_h, tile_w, bins, m,
                                         float(tau), C.byref(o), fptr, C.byref(pr)))
    try:
        n = int(pr.count)
        res = JoinResult(
            np.ctypeslib.as_array(pr.left, shape=(n,)).copy() if n else np.empty(0, np.int32),
            np.ctypeslib.as_array(pr.right, shape=(n,)).copy() if n else np.empty(0, np.int32),
            np.ctypeslib.as_array(pr.dist, shape=(n,)).copy() if n else np.empty(0, np.float32))
    finally:
        capi.lib().pdb_pairs_free(C.byref(pr))
    return (feats, res) if want_features else res


# ---------------------------------------------------------------------------
# Object API (include/patchdb/core.hpp, etl.hpp, query.hpp)


@dataclass
class BoundingBox:
    x1: int = 0
    y1: int = 0
    x2: int = 0
    y2: int = 0

    def width(self) -> int:
        return self.x2 - self.x1

    def height(self) -> int:
        return self.y2 - self.y1

    def valid(self) -> bool:
        return self.x1 < self.x2 and self.y1 < self.y2


@dataclass
class Frame:
    """uint8 row-major HWC interleaved RGB frame (core.hpp:66-80)."""
    video_id: str
    frame_no: int
    pixels: np.ndarray  # [H, W, 3] uint8

    @property
    def width(self) -> int:
        return int(self.pixels.shape[1])

    @property
    def height(self) -> int:
        return int(self.pixels.shape[0])


@dataclass
class LineageStep:
    op_name: str
    source: object          # (video_id, frame_no) or parent patch id
    region: Optional[BoundingBox] = None
    params_digest: int = 0


@dataclass
class Patch:
    """core.hpp:121-141: id, lineage (most recent first), float data, shape, metadata."""
    patch_id: int
    data: np.ndarray
    shape: Tuple[int, ...]
    meta: dict = field(default_factory=dict)
    lineage: List[LineageStep] = field(default_factory=list)

    def is_pixel(self) -> bool:
        return len(self.shape) == 3 and self.shape[2] == 3

    def is_feature(self) -> bool:
        return len(self.shape) == 1


class _Ids:
    """The global patch-id counter (src/core.cpp:9,31)."""
    next_id = 1


def reset_patch_ids(start: int = 1) -> None:
    _Ids.next_id = start


def next_patch_id() -> int:
    v = _Ids.next_id
    _Ids.next_id += 1
    return v


def _fnv_digest(name: str, items: Sequence[Tuple[str, object]]) -> int:
    """ParamsDigest (include/patchdb/core.hpp:155-196): FNV-1a-64 over the
    big-endian byte record str8(op_name) then, per param, str8(key) and
    either tag 0 + i64 (int), tag 1 + the f64 bit pattern (float) or tag 2
    + str16 (string)."""
    import struct
    buf = bytearray()
    nb = name.encode()
    buf += bytes([len(nb)]) + nb
    for k, v in items:
        kb = k.encode()
        if isinstance(v, float):
            buf += bytes([len(kb)]) + kb + b"\x01" + struct.pack(">d", v)
        elif isinstance(v, str):
            vb = v.encode()
            buf += bytes([len(kb)]) + kb + b"\x02" + struct.pack(">H", len(vb)) + vb
        else:
            buf += bytes([len(kb)]) + kb + b"\x00" + int(v & 0xFFFFFFFFFFFFFFFF).to_bytes(8, "big")
    h = 0xCBF29CE484222325
    for x in buf:
        h ^= x
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


@dataclass
class GeneratorSpec:
    kind: str = "whole_image"   # whole_image | tiles (blob/glyph are out of scope)
    tile_w: int = 0
    tile_h: int = 0

    def validate(self) -> None:
        if self.kind == "tiles":
            if self.tile_w < 1 or self.tile_h < 1:
                raise ConfigError("tiles generator needs tile_w and tile_h >= 1")
        elif self.kind != "whole_image":
            raise ConfigError(f"unknown generator kind '{self.kind}'")


@dataclass
class TransformerSpec:
    kind: str = "color_histogram"
    bins: int = 8
    mode: str = "per_channel"   # "joint" is the BASELINE 4x4x4 extension

    def validate(self) -> None:
        if self.kind != "color_histogram":
            raise ConfigError(f"unknown transformer kind '{self.kind}'")
        if self.bins < 2:
            raise ConfigError("color_histogram needs at least 2 bins per channel")


def make_patch(frame: Frame, box: BoundingBox) -> Patch:
    """src/core.cpp:78-113 (the float crop is a zero-copy view here; the
    fused K1 path never materialises it)."""
    if not box.valid() or box.x2 > frame.width or box.y2 > frame.height:
        raise RegionOutOfBoundsError(
            f"region ({box.x1},{box.y1},{box.x2},{box.y2}) exceeds frame "
            f"{frame.width}x{frame.height}")
    pid = next_patch_id()
    crop = frame.pixels[box.y1:box.y2, box.x1:box.x2, :]
    digest = _fnv_digest("make_patch", [("x1", box.x1), ("y1", box.y1), ("x2", box.x2),
                                        ("y2", box.y2)])
    step = LineageStep("make_patch", (frame.video_id, frame.frame_no), box, digest)
    meta = {"frameno": frame.frame_no, "bbox": (box.x1, box.y1, box.x2, box.y2),
            "frame_w": frame.width, "frame_h": frame.height}
    return Patch(pid, crop, (box.height(), box.width(), 3), meta, [step])


def generate(frames: Iterable[Frame], g: GeneratorSpec) -> Iterator[Patch]:
    """src/etl.cpp:252-298: whole_image or floor-grid tiles, row by row, tx fastest."""
    g.validate()
    for f in frames:
        if g.kind == "whole_image":
            yield make_patch(f, BoundingBox(0, 0, f.width, f.height))
            continue
        ntx, nty = f.width // g.tile_w, f.height // g.tile_h
        for ty in range(nty):
            for tx in range(ntx):
                yield make_patch(f, BoundingBox(tx * g.tile_w, ty * g.tile_h,
                                                (tx + 1) * g.tile_w, (ty + 1) * g.tile_h))


def _derive(parent: Patch, hist: np.ndarray, t: TransformerSpec) -> Patch:
    digest = _fnv_digest("color_histogram", [("bins", t.bins)])
    step = LineageStep("color_histogram", parent.patch_id, None, digest)
    return Patch(next_patch_id(), hist, (hist.shape[0],), dict(parent.meta),
                 [step] + list(parent.lineage))


def apply_transformer(p: Patch, t: TransformerSpec) -> Patch:
    """src/etl.cpp:330-354 on the GPU (K1, float-patch entry point)."""
    t.validate()
    if not p.is_pixel():
        raise ShapeError(f"transformer input must be pixel shaped [h,w,3], patch {p.patch_id} is not")
    px = np.ascontiguousarray(p.data, dtype=np.float32).reshape(1, p.shape[0], p.shape[1], 3)
    hist = color_histogram(px, t.bins, t.mode)[0]
    return _derive(p, hist, t)


def transform(patches: Iterable[Patch], t: TransformerSpec, batch: int = 4096) -> Iterator[Patch]:
    """src/etl.cpp:364-373, batched: pixel patches of one shape are grouped into
    one K1 launch.  Ids are assigned in the reference's interleaved order
    (each derived patch takes its id right after its parent's)."""
    t.validate()
    it = iter(patches)
    while True:
        chunk = []
        for p in it:
            chunk.append(p)
            if len(chunk) == batch:
                break
        if not chunk:
            return
        for p in chunk:
            if not p.is_pixel():
                raise ShapeError(
                    f"transformer input must be pixel shaped [h,w,3], patch {p.patch_id} is not")
        shapes = {p.shape for p in chunk}
        hists = {}
        for shp in shapes:
            idx = [k for k, p in enumerate(chunk) if p.shape == shp]
            px = np.stack([np.asarray(chunk[k].data, dtype=np.float32) for k in idx])
            h = color_histogram(px, t.bins, t.mode)
            for r, k in enumerate(idx):
                hists[k] = h[r]
        for k, p in enumerate(chunk):
            yield _derive(p, hists[k], t)


class BuildSide(enum.IntEnum):
    automatic = 0
    left = 1
    right = 2


def _checked_dim(items: Sequence[Patch]) -> int:
    """src/query.cpp:467-477."""
    d = int(np.asarray(items[0].data).size) if items else 0
    if items and d == 0:
        raise ShapeError("similarity join needs non-empty patch data")
    for p in items:
        if int(np.asarray(p.data).size) != d:
            raise MixedDimensionError(
                f"similarity join saw {d} and {int(np.asarray(p.data).size)} dimensional patches")
    return d


def sim_join_pairs(left: Sequence[Patch], right: Sequence[Patch], tau: float,
                   side: BuildSide = BuildSide.automatic,
                   probes: Optional[list] = None) -> List[Tuple[Patch, Patch]]:
    """src/query.cpp:1094-1104 (run_sim_join 485-528) on the B200 join.

    Pairs come out in the reference's order: probe order, then ascending
    build-side patch id; ``probes`` (a list) receives the probe-row count.
    """
    if tau < 0.0:
        raise ConfigError("similarity join needs tau >= 0")
    chosen = side if side != BuildSide.automatic else (
        BuildSide.left if len(left) <= len(right) else BuildSide.right)
    dl, dr = _checked_dim(left), _checked_dim(right)
    if left and right and dl != dr:
        raise DimensionMismatchError(f"similarity join over {dl} and {dr} dimensional sides")
    if not left or not right:
        if probes is not None:
            probes[:] = [0]
        return []
    build = left if chosen == BuildSide.left else right
    ids = [p.patch_id for p in build]
    if len(set(ids)) != len(ids):
        seen = set()
        for i in ids:
            if i in seen:
                raise DuplicatePatchIdError(f"patch id {i} appears twice on the build side")
            seen.add(i)
    Lm = np.stack([np.asarray(p.data, dtype=np.float32).ravel() for p in left])
    Rm = np.stack([np.asarray(p.data, dtype=np.float32).ravel() for p in right])
    res = sim_join(Lm, Rm, tau, sort=False)
    li, ri = res.left.astype(np.int64), res.right.astype(np.int64)
    if chosen == BuildSide.left:
        bid = np.array([left[k].patch_id for k in range(len(left))], dtype=np.uint64)[li]
        order = np.lexsort((bid, ri))   # probe = right position, then build id
    else:
        bid = np.array([right[k].patch_id for k in range(len(right))], dtype=np.uint64)[ri]
        order = np.lexsort((bid, li))
    if probes is not None:
        probes[:] = [len(right) if chosen == BuildSide.left else len(left)]
    return [(left[int(li[k])], right[int(ri[k])]) for k in order]


# ---------------------------------------------------------------------------
# Near-duplicate grouping (run_dedup, src/query.cpp:535-566) on the tau-graph
# of the B200 join (csrc/dedup.cu).


class DedupGroups:
    """run_dedup's result: representatives (kept order) and, per
    representative, its members in arrival order (built on first use);
    rep_of[i] is item i's representative."""

    def __init__(self, reps: np.ndarray, rep_of: np.ndarray):
        self.reps = reps
        self.rep_of = rep_of
        self._members = None

    @property
    def members(self) -> List[np.ndarray]:
        if self._members is None:
            n = self.rep_of.shape[0]
            order = np.argsort(self.rep_of, kind="stable")  # members keep arrival order
            bounds = np.searchsorted(self.rep_of[order], self.reps)
            self._members = np.split(order, bounds[1:]) if n else []
        return self._members


def dedup(X: np.ndarray, tau: float) -> DedupGroups:
    """Host rows [n, d] fp32 -> DedupGroups (the C-ABI's pdb_dedup)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n = X.shape[0]
    d = X.shape[1] if X.ndim == 2 else 0
    rep_of = np.empty(max(n, 1), dtype=np.int64)
    nr = C.c_int64()
    _check(capi.lib().pdb_dedup(capi.ptr(X), n, d, float(tau), None, capi.ptr(rep_of),
                                C.byref(nr)))
    rep_of = rep_of[:n]
    return DedupGroups(np.flatnonzero(rep_of == np.arange(n)), rep_of)


def dedup_device(X, tau: float, stream=None):
    """Device rows (CUDA fp32 tensor [n, d]) -> (rep_of int64 tensor, n_reps)."""
    import torch
    assert X.is_cuda and X.dtype == torch.float32 and X.is_contiguous()
    n, d = int(X.shape[0]), int(X.shape[1])
    rep_of = torch.empty(max(n, 1), dtype=torch.int64, device=X.device)
    s = stream if stream is not None else torch.cuda.current_stream(X.device)
    o = capi.JoinOpts()
    o.stream = C.c_void_p(s.cuda_stream)
    nr = C.c_int64()
    _check(capi.lib().pdb_dedup_dev(X.data_ptr(), n, d, float(tau), C.byref(o),
                                    rep_of.data_ptr(), C.byref(nr)))
    return rep_of[:n], int(nr.value)


def _dedup_matrix(items: Sequence[Patch], what: str) -> np.ndarray:
    d = int(np.asarray(items[0].data).size)
    if d == 0:
        raise ShapeError(f"{what} needs non-empty patch data")
    for p in items:
        if int(np.asarray(p.data).size) != d:
            raise MixedDimensionError(
                f"{what} saw {d} and {int(np.asarray(p.data).size)} dimensional patches")
    return np.stack([np.asarray(p.data, dtype=np.float32).ravel() for p in items])


def dedup_groups(items: Sequence[Patch], tau: float) -> List[Patch]:
    """PlanNode::dedup's output (src/query.cpp:860-880, make_group_patch
    568-582): one derived patch per representative, in kept order, with
    metadata group_labels (sorted distinct string labels of the members)
    and group_size."""
    if tau < 0.0:
        raise ConfigError("dedup needs tau >= 0")
    if not items:
        return []
    g = dedup(_dedup_matrix(items, "dedup"), tau)
    digest = _fnv_digest("dedup_group", [("tau", float(tau))])
    out = []
    for r, mem in zip(g.reps, g.members):
        rep = items[int(r)]
        labels = sorted({items[int(m)].meta["label"] for m in mem
                         if isinstance(items[int(m)].meta.get("label"), str)})
        meta = dict(rep.meta)
        meta["group_labels"] = labels
        meta["group_size"] = int(len(mem))
        step = LineageStep("dedup_group", rep.patch_id, None, digest)
        out.append(Patch(next_patch_id(), np.asarray(rep.data), tuple(rep.shape), meta,
                         [step] + list(rep.lineage)))
    return out


def dedup_stream(items: Iterable[Patch], tau: float) -> Iterator[Patch]:
    """dedup_stream (src/query.cpp:1063-1092): the kept patches, in order.
    The B200 build drains its input first (the scan is global)."""
    if tau < 0.0:
        raise ConfigError("dedup needs tau >= 0")
    items = list(items)
    if not items:
        return iter(())
    for p in items:
        if np.asarray(p.data).size == 0:
            raise ShapeError("dedup needs non-empty patch data")
    g = dedup(_dedup_matrix(items, "dedup"), tau)
    return iter([items[int(r)] for r in g.reps])


# ---------------------------------------------------------------------------
# Plans routed onto the join.


def nl_join_within(left: Sequence[Patch], right: Sequence[Patch],
                   radius: float) -> List[Tuple[Patch, Patch]]:
    """PlanNode::nl_join(left, right, within_of(0, 1, radius)) over
    single-patch tuples (src/query.cpp:142-151, 705-744): every (l, r) with
    euclidean(l, r) <= radius, in nested-loop order (left order, then right
    order) -- the B200 cross join sorted by (left, right).  A dimension
    mismatch raises DimensionMismatchError as the predicate's first
    evaluation would; empty sides give no tuples."""
    if not left or not right:
        return []
    dims = {int(np.asarray(p.data).size) for p in left} | {int(np.asarray(p.data).size)
                                                            for p in right}
    if len(dims) != 1:
        a, b = sorted(dims)[:2]
        raise DimensionMismatchError(f"distance between {a} and {b} dimensional patches")
    Lm = np.stack([np.asarray(p.data, dtype=np.float32).ravel() for p in left])
    Rm = np.stack([np.asarray(p.data, dtype=np.float32).ravel() for p in right])
    if Lm.shape[1] == 0:
        # zero-dimensional patches are all at distance 0
        return [(l, r) for l in left for r in right] if radius >= 0 else []
    if radius < 0:
        return []
    res = sim_join(Lm, Rm, radius, sort=True)
    return [(left[int(i)], right[int(j)]) for i, j in zip(res.left, res.right)]


def q1_duplicate_frames(frames: np.ndarray, bins: int, tau: float):
    """The q1 near-duplicate-frame query (src/bench.cpp:695-730) on frames
    numbered 0..F-1: whole-image colour histograms (K1, generate whole_image
    + color_histogram), then select(sim_join(h, h, tau), frameno != frameno)
    (K2 + K3).  Returns (frame a, frame b) of every result tuple in the
    reference's emission order: sim_join's probe order (the right side,
    build side left on the size tie), then ascending build id."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    F, H, W = frames.shape[:3]
    h = featurize_tiles(frames, H, W, bins, "per_channel")
    res = sim_join(h, None, tau, self_join=True, sort=False)
    i = res.left.astype(np.int64)
    j = res.right.astype(np.int64)
    a = np.concatenate([i, j])
    b = np.concatenate([j, i])
    order = np.lexsort((a, b))
    return a[order], b[order]


# ---------------------------------------------------------------------------
# Frame source: the reference's VideoStore files.


class VideoStore:
    """VideoStore::open / scan (include/patchdb/storage.hpp:60-89) over the
    reference's store files, decoded by libpdb_cuda's reader (parallel zlib
    clip decode on host threads); ``featurize`` feeds the frames to K1."""

    def __init__(self, handle, info):
        self._h = handle
        self.info = info

    @classmethod
    def open(cls, path: str) -> "VideoStore":
        h = C.c_void_p()
        _check(capi.lib().pdb_store_open(str(path).encode(), C.byref(h)))
        info = capi.StoreInfo()
        _check(capi.lib().pdb_store_describe(h, C.byref(info)))
        return cls(h, info)

    def close(self) -> None:
        if getattr(self, "_h", None) and capi is not None:
            capi.lib().pdb_store_close(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def frame_count(self) -> int:
        return int(self.info.frame_count)

    @property
    def width(self) -> int:
        return int(self.info.width)

    @property
    def height(self) -> int:
        return int(self.info.height)

    @property
    def video_id(self) -> str:
        return self.info.video_id.decode()

    def _range(self, rng):
        if rng is None:
            return -1, -1, self.frame_count
        lo, hi = int(rng[0]), int(rng[1])
        if lo >= hi:
            raise ConfigError("scan range low bound must be below high bound")
        n = max(min(hi, self.frame_count) - min(lo, self.frame_count), 0)
        return lo, hi, n  # the library clamps both ends

    def scan_array(self, rng: Optional[Tuple[int, int]] = None, threads: int = 0) -> np.ndarray:
        """Frames [lo, hi) as a [n, H, W, 3] uint8 array (scan's frames)."""
        lo, hi, n = self._range(rng)
        out = np.empty((max(n, 1), self.height, self.width, 3), np.uint8)
        got = C.c_int64()
        _check(capi.lib().pdb_store_read(self._h, lo, hi, capi.ptr(out), C.byref(got),
                                         threads or _host_threads()))
        return out[:got.value]

    def scan(self, rng: Optional[Tuple[int, int]] = None) -> Iterator[Frame]:
        """VideoStore::scan: Frame objects in ascending frame order."""
        arr = self.scan_array(rng)
        first = 0 if rng is None else min(int(rng[0]), self.frame_count)
        for k in range(arr.shape[0]):
            yield Frame(self.video_id, first + k, arr[k])

    def featurize(self, tile_h: int, tile_w: int, bins: int = 8, mode="per_channel",
                  rng: Optional[Tuple[int, int]] = None, threads: int = 0, stream=None):
        """Decode + K1 chunk by chunk: device features [frames * tiles, D]."""
        import torch
        m = _mode(mode)
        lo, hi, n = self._range(rng)
        D = hist_dim(bins, m)
        tiles = (self.width // tile_w) * (self.height // tile_h)
        out = torch.empty((max(n, 1) * tiles, D), dtype=torch.float32, device="cuda")
        s = stream if stream is not None else torch.cuda.current_stream()
        got = C.c_int64()
        _check(capi.lib().pdb_store_featurize(self._h, lo, hi, tile_h, tile_w, bins, m,
                                              out.data_ptr(), C.byref(got),
                                              threads or _host_threads(),
                                              C.c_void_p(s.cuda_stream)))
        return out[:got.value * tiles]


def _host_threads() -> int:
    import os
    return max(1, min(os.cpu_count() or 1, 64))

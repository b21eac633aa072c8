"""Host-side multi-GPU plumbing for the hot path (one process per GPU,
torch.distributed over NCCL on the box, gloo in the CPU tests).

The reference is single-threaded with no distributed backend (SPEC.md:495,
565); the sharding here is the B200 build's own:

* featurization: frames are independent -> contiguous frame ranges per rank;
  every rank joins against all the features (config 2: 64,000 x 64 x 4 =
  16 MB).  With PeerFeatures the exchange is fused into K1: each rank maps
  every rank's feature matrix over CUDA IPC and writes its slice into all of
  them with P2P stores over NVLink while it counts, so one on-stream barrier
  replaces the all-gather (all_gather_rows is the NCCL fallback);
* cross join (config 3): L is row-sharded in contiguous ranges
  (left_rows) and R is broadcast once over NCCL; each rank runs a plain
  cross join of its rows, so the L side of the band plan is divided by the
  rank count and only R's side is replicated (the broadcast relation);
* self-join: the 128-row blocks of L in boustrophedon rounds -- block
  k*world + (rank if k even else world-1-rank) (pdb_join_opts
  shard_index/shard_count) -- which balances the triangular self-join and
  skewed clusters without a scheduler; pairs stay on the rank
  that found them (indices are global), counts are all-reduced, and
  gather_pairs() collects them on one rank when a caller wants them there.
"""

from __future__ import annotations

import numpy as np

BM = 128  # rows per block of L in the screen kernel (join.cu BM)


def frame_range(rank: int, world: int, n_frames: int):
    return n_frames * rank // world, n_frames * (rank + 1) // world


def left_rows(rank: int, world: int, n_left: int):
    """Cross joins (config 3): rank's contiguous range [l0, l1) of L.  The
    rank joins L[l0:l1] against all of R as a plain cross join (its band
    plan covers only its own rows); its pairs' left indices shift by l0."""
    return n_left * rank // world, n_left * (rank + 1) // world


def row_blocks(rank: int, world: int, n_rows: int):
    nb = (n_rows + BM - 1) // BM
    k = np.arange((nb + world - 1) // world, dtype=np.int64)
    b = k * world + np.where(k & 1, world - 1 - rank, rank)
    return b[b < nb]


def shard_rows(rank: int, world: int, n_rows: int) -> np.ndarray:
    """Row indices of L scanned by `rank` (what pdb_sim_join_dev does with
    shard_index=rank, shard_count=world)."""
    rows = (row_blocks(rank, world, n_rows)[:, None] * BM + np.arange(BM)[None]).ravel()
    return rows[rows < n_rows]


def selfjoin_tiles(rank: int, world: int, n_rows: int, bn: int = 256) -> int:
    """Screen tiles rank executes in a self-join (upper triangle by 256-col tiles)."""
    nt = (n_rows + bn - 1) // bn
    return int(sum(nt - (b >> 1) for b in row_blocks(rank, world, n_rows)))


class PeerFeatures:
    """Every rank's feature matrix mapped into this process (CUDA IPC), for
    pdb_featurize_tiles_dev_multi: `ptrs(offset_elems)` lists the local
    buffer first, then each peer's, all shifted by `offset_elems` floats.
    The mapped storages stay referenced for the object's lifetime."""

    def __init__(self, feats, group=None):
        import torch.distributed as dist
        import torch
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.elem = feats.element_size()
        mine = (feats.untyped_storage()._share_cuda_(), feats.storage_offset())
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._keep = []
        self._base = []
        for r, (h, off) in enumerate(allh):
            if r == self.rank:
                self._base.append(feats.data_ptr())
                continue
            st = torch.UntypedStorage._new_shared_cuda(*h)
            self._keep.append(st)
            self._base.append(st.data_ptr() + off * self.elem)
        # local first
        self._order = [self.rank] + [r for r in range(self.world) if r != self.rank]

    def ptrs(self, offset_elems: int):
        return [self._base[r] + offset_elems * self.elem for r in self._order]


def all_gather_rows(local, world: int, group=None):
    """Concatenate equally sized per-rank row blocks on every rank."""
    import torch
    import torch.distributed as dist
    out = torch.empty((local.shape[0] * world,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    if world == 1:
        out.copy_(local)
        return out
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


def gather_pairs(left, right, dist_, world: int, dst: int = 0, group=None):
    """Collect every rank's (left, right, dist) on rank `dst` (others get
    None): counts are all-gathered first, then the padded arrays."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return left, right, dist_
    n = torch.tensor([left.shape[0]], dtype=torch.int64, device=left.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts) if counts else 0
    pack = torch.zeros((3, m), dtype=torch.float64, device=left.device)
    pack[0, :left.shape[0]] = left.double()
    pack[1, :left.shape[0]] = right.double()
    pack[2, :left.shape[0]] = dist_.double()
    bufs = [torch.empty_like(pack) for _ in range(world)]
    dist.all_gather(bufs, pack, group=group)
    if dist.get_rank(group) != dst:
        return None
    l = torch.cat([b[0, :c] for b, c in zip(bufs, counts)]).to(torch.int32)
    r = torch.cat([b[1, :c] for b, c in zip(bufs, counts)]).to(torch.int32)
    d = torch.cat([b[2, :c] for b, c in zip(bufs, counts)]).to(torch.float32)
    return l, r, d

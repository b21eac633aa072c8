"""Multi-process (world_size 2, gloo, CPU) test of the host-side sharding:
frame ranges, the feature all-gather, the cyclic row-block split of the join
and the pair gather reproduce the single-process result exactly.  The CPU
oracle stands in for K1/K2 here (no GPU in this container); on the box the
same plumbing carries the CUDA results (bench.py, NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_07607_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1812_07607_b200 import workloads
        F, H, W = 10, 96, 128
        f0, f1 = shard.frame_range(rank, world, F)
        fr, _ = workloads.frames(f1 - f0, H, W, seed=2, first=f0)
        feats = torch.from_numpy(oracle.featurize_tiles(fr, 24, 32, 4, 1))
        allf = shard.all_gather_rows(feats, world).numpy()
        rows = shard.shard_rows(rank, world, allf.shape[0])
        ls, rs, ds = [], [], []
        for b in shard.row_blocks(rank, world, allf.shape[0]):
            r0, r1 = int(b) * shard.BM, min(int(b + 1) * shard.BM, allf.shape[0])
            l, r, d = oracle.sim_join(allf, None, 0.05, self_join=True, rows=(r0, r1), threads=1)
            ls.append(l), rs.append(r), ds.append(d)
        l = torch.from_numpy(np.concatenate(ls))
        r = torch.from_numpy(np.concatenate(rs))
        d = torch.from_numpy(np.concatenate(ds).astype(np.float32))
        assert np.isin(l.numpy(), rows).all()
        got = shard.gather_pairs(l, r, d, world)
        if rank == 0:
            q.put((allf, got[0].numpy(), got[1].numpy(), got[2].numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_featurize_gather_join():
    from oracle import oracle
    from paper_1812_07607_b200 import workloads
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allf, l, r, d = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    fr, _ = workloads.frames(10, 96, 128, seed=2)
    want_f = oracle.featurize_tiles(fr, 24, 32, 4, 1)
    assert np.array_equal(allf, want_f)
    ol, orr, od = oracle.sim_join(want_f, None, 0.05, self_join=True)
    k = np.lexsort((r, l))
    assert np.array_equal(l[k], ol) and np.array_equal(r[k], orr)
    assert np.array_equal(d[k], od.astype(np.float32))


def test_row_block_partition_and_balance():
    n = 64000
    seen = np.concatenate([shard.shard_rows(k, 8, n) for k in range(8)])
    assert np.array_equal(np.sort(seen), np.arange(n))
    tiles = [shard.selfjoin_tiles(k, 8, n) for k in range(8)]
    assert max(tiles) / min(tiles) < 1.02   # cyclic blocks balance the triangle
    assert shard.frame_range(7, 8, 1000) == (875, 1000)


def _cross_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1812_07607_b200 import workloads
        L, R, pl, pr = workloads.config3(n=6000)
        # R travels from rank 0 (the broadcast relation); L rows are local
        Rt = torch.from_numpy(R) if rank == 0 else torch.empty(R.shape, dtype=torch.float32)
        dist.broadcast(Rt, src=0)
        l0, l1 = shard.left_rows(rank, world, L.shape[0])
        l, r, d = oracle.sim_join(L[l0:l1], Rt.numpy(), 0.02, threads=1)
        got = shard.gather_pairs(torch.from_numpy(l.astype(np.int64) + l0).to(torch.int32),
                                 torch.from_numpy(r), torch.from_numpy(d.astype(np.float32)), world)
        if rank == 0:
            q.put(tuple(t.numpy() for t in got))
    finally:
        dist.destroy_process_group()


def test_two_rank_row_sharded_cross_join():
    """Config 3's multi-GPU layout (L row-sharded, R broadcast): the union of
    the ranks' pairs, shifted to global rows, is the single-process join."""
    from oracle import oracle
    from paper_1812_07607_b200 import workloads
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cross_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    l, r, d = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    L, R, pl, pr = workloads.config3(n=6000)
    ol, orr, od = oracle.sim_join(L, R, 0.02)
    k = np.lexsort((r, l))
    assert np.array_equal(l[k], ol) and np.array_equal(r[k], orr)
    assert np.array_equal(d[k], od.astype(np.float32))
    assert len(ol) >= len(pl) > 0
    assert shard.left_rows(1, 2, 6000) == (3000, 6000)

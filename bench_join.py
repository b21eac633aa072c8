"""Join-only benchmark lines for BASELINE.json's configs 1, 3, 4 and 5
(``python bench.py --workload c1|c3|c4|c5``; the default bench line is
config 2, the featurize -> join pipeline).

One step = one full threshold join of the configured relations, device
resident (``pdb_sim_join_dev`` / ``pdb_cosine_join_bf16_dev``), L2 flushed
before each step.  ``value`` is candidate pairs per second over the whole
job (N(N-1)/2 for a self-join, nL*nR for a cross join: the GPU is not
credited for the lower triangle it skips), in Gpairs/s.  ``e2e`` is the same
join through the host C-ABI call (pinned host relations in, host pairs out).

Multi-GPU (torchrun, one process per GPU): rank 0 generates the relations
and broadcasts them once over NCCL (timed separately as ``setup``); every
rank then scans its boustrophedon share of L's 128-row blocks against all of
R (``pdb_join_opts.shard_*``), pairs stay on the rank that found them and
the pair counts are all-reduced.  Strong scaling: the join is fixed.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import statistics
import time

import numpy as np

JOINS = {
    "c1": dict(workload="config1_selfjoin: 20,000 x 64 fp32, 200 Gaussian clusters (sigma 0.02), "
                        "L1-normalised, seed 0; L2 self-join eps=0.05, (i<j) pairs",
               kind="l2", self_join=True, tau=0.05),
    "c3": dict(workload="config3_cross: 1,048,576 x 1,048,576 fp32 d=128, 10,000-cluster mixture "
                        "(sigma 0.01), 0.5% planted near-duplicates (sigma 1e-3), seed 3; "
                        "L2 join eps=0.02, L row-sharded",
               kind="l2", self_join=False, tau=0.02),
    "c4": dict(workload="config4_cosine: 200,000 x 2048 bf16 normalize(ReLU(P z)), seed 4, "
                        "0.5% planted near-duplicates; cosine self-join >= 0.95",
               kind="cos", self_join=True, tau=0.95),
    "c5": dict(workload="config5_skewed: 4,194,304 x 64 fp32, 20% in 50 simplex clusters "
                        "(sigma 1e-3), 80% Dirichlet(1), seed 5; L2 self-join eps=0.01",
               kind="l2", self_join=True, tau=0.01),
    "dedup": dict(workload="dedup of the config-2 tile histograms: 64,000 x 64 joint 4x4x4 "
                           "histograms of 1000 synthetic 480x640 frames (seed 2), tau=0.05 "
                           "(run_dedup / PlanNode::dedup semantics)",
                  kind="dedup", self_join=True, tau=0.05),
}


def _gen(which):
    from paper_1812_07607_b200 import workloads
    if which == "c1":
        return workloads.config1(), None
    if which == "c3":
        L, R, _, _ = workloads.config3()
        return L, R
    if which == "c4":
        return workloads.bf16_bits(workloads.config4(device="cuda")), None
    if which == "c5":
        return workloads.config5(), None
    if which == "dedup":
        from paper_1812_07607_b200 import patchdb
        import torch
        fr, _ = workloads.frames(1000, 480, 640, seed=2)
        feats = patchdb.featurize_tiles(torch.from_numpy(fr).cuda(), 60, 80, 4, "joint")
        return feats.cpu().numpy(), None
    raise ValueError(which)


def _cpu_baseline(which, L, R, cfg, threads):
    """The reference (oracle/_ref, ball tree build + balltree_within probes)
    for the L2 configs, the C restatement for the restated cosine config, on
    a bounded random sample of probe rows, extrapolated to the full join."""
    from oracle import oracle
    rng = np.random.default_rng(1)
    n = L.shape[0]
    cand = n * (n - 1) / 2 if cfg["self_join"] else n * R.shape[0]
    if cfg["kind"] == "dedup":
        k = int(os.environ.get("PDB_REF_DEDUP_ROWS", 16000))
        sub = np.ascontiguousarray(L[:k])
        t0 = time.perf_counter()
        oracle.ref_dedup(sub, cfg["tau"])
        t_s = time.perf_counter() - t0
        # run_dedup's cost grows with n * reps (attach scans every kept rep):
        # extrapolate quadratically from the prefix sample
        t = t_s * (n / sub.shape[0]) ** 2
        return {"value": n / t, "unit": "items/s", "cores": 1, "kind": "reference",
                "sample": f"reference PlanNode::dedup (oracle/_ref, run_dedup) on the first {k} "
                          f"items ({t_s:.2f} s, single-threaded as the reference is), "
                          f"extrapolated quadratically to {n}",
                "extrapolated_s": t}
    if cfg["kind"] == "l2":
        rows = int(os.environ.get("PDB_REF_PROBE_ROWS", {"c1": 2048, "c3": 512, "c5": 512}[which]))
        idx = np.sort(rng.choice(n, size=min(rows, n), replace=False))
        sub = np.ascontiguousarray(L[idx])
        Rf = L if cfg["self_join"] else R
        _, t_build, t_probe = oracle.ref_join_probe_timed(sub, Rf, cfg["tau"], False, 0,
                                                          sub.shape[0], threads)
        t = t_build + t_probe * n / sub.shape[0]
        kind = "reference"
        sample = (f"reference build_balltree({Rf.shape[0]}) + balltree_within for {sub.shape[0]} "
                  f"random probe rows on {threads} threads (build {t_build:.2f} s, probes "
                  f"{t_probe:.2f} s), extrapolated to {n} probes")
    else:
        rows = int(os.environ.get("PDB_REF_PROBE_ROWS", 64))
        t0 = time.perf_counter()
        oracle.cosine_join_bf16(L, None, cfg["tau"], self_join=True, rows=(0, rows),
                                threads=threads)
        t_s = time.perf_counter() - t0
        # rows i < rows of the upper triangle: sum_{i<rows} (n-1-i) pairs
        done = rows * (n - 1) - rows * (rows - 1) / 2
        t = t_s * cand / done
        kind = "port"
        sample = (f"C restatement (oracle/pdb_oracle.c orc_cosine_join_bf16, fp64) on probe rows "
                  f"0..{rows - 1} ({done:.3g} of {cand:.3g} pairs, {t_s:.2f} s) on {threads} "
                  f"threads, extrapolated")
    return {"value": cand / t / 1e9, "unit": "Gpairs/s", "cores": threads, "kind": kind,
            "sample": sample, "extrapolated_s": t}


def run_reference(args, rank, world, which, metric):
    if rank != 0:
        return 0
    cfg = JOINS[which]
    if which == "c4":  # the generator runs on torch; keep it on the CPU in this arm
        from paper_1812_07607_b200 import workloads
        L, R = workloads.bf16_bits(workloads.config4(device="cpu")), None
    else:
        L, R = _gen(which)
    threads = os.cpu_count() or 1
    vals = []
    base = None
    for k in range(args.warmup + args.steps):
        base = _cpu_baseline(which, L, R, cfg, threads)
        if k >= args.warmup:
            vals.append(base["value"])
    v = statistics.mean(vals)
    base["value"] = v
    n = L.shape[0]
    cand = n * (n - 1) / 2 if cfg["self_join"] else n * R.shape[0]
    print(json.dumps({
        "impl": "reference", "metric": metric, "value": v, "unit": "Gpairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cand / (v * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if cfg["kind"] == "l2" else "bf16/f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": n, "candidate_pairs": cand},
        "cpu_baseline": base,
        "e2e": {"value": v, "unit": "Gpairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def run_ours(args, rank, world, local_rank, which, metric, peaks, clock_sampler):
    line = measure(args, rank, world, local_rank, which, metric, peaks, clock_sampler)
    if rank == 0:
        print(json.dumps(line))
    return 0


def _verify_c3(Lh, Rh, planted, gl, gr, threads):
    """Config 3's cpu_baseline leg: the reference
    itself (oracle/_ref: build_balltree over R + balltree_within) on S probe
    rows -- 256 strided over L plus 64 planted rows -- timed and compared
    with the GPU pairs of those rows; plus every planted pair in the GPU
    output.  Returns (cpu_baseline dict, checked dict)."""
    from oracle import oracle
    n = Lh.shape[0]
    pl, pr = planted
    rows = np.unique(np.concatenate([np.arange(0, n, n // 256), pl[:: max(1, len(pl) // 64)]]))
    rl, rr, t_build, t_probe = oracle.ref_join_probe_pairs(Lh[rows], Rh, 0.02, threads)
    want = np.stack([rows[rl], rr], 1)
    flag = np.zeros(n, bool)
    flag[rows] = True
    m = flag[gl]
    got = np.stack([gl[m], gr[m]], 1)
    got = got[np.lexsort((got[:, 1], got[:, 0]))]
    rows_equal = bool(np.array_equal(got, want))
    keys = set((gl.astype(np.int64) << 32 | gr.astype(np.int64)).tolist())
    found = sum(1 for a, b in zip(pl.tolist(), pr.tolist()) if (a << 32 | b) in keys)
    cand = float(n) * Rh.shape[0]
    t = t_build + t_probe * n / rows.shape[0]
    base = {"value": cand / t / 1e9, "unit": "Gpairs/s", "cores": threads, "kind": "reference",
            "sample": f"reference build_balltree({Rh.shape[0]}) + balltree_within for "
                      f"{rows.shape[0]} probe rows (256 strided + 64 planted) on {threads} "
                      f"threads (build {t_build:.2f} s, probes {t_probe:.2f} s), probes "
                      f"extrapolated to {n}",
            "extrapolated_s": t}
    checked = {"rows": int(rows.shape[0]), "pairs_in_rows": int(len(want)),
               "rows_equal_reference": rows_equal, "planted": int(len(pl)),
               "planted_found": int(found),
               "oracle": "the reference's own sim_join probe (oracle/_ref) on those rows; the "
                         "whole pair set is checked against the exact CPU join in "
                         "tests/test_fullsize_gpu.py"}
    return base, checked


def measure(args, rank, world, local_rank, which, metric, peaks, clock_sampler, dense=False):
    import torch
    import torch.distributed as dist

    from paper_1812_07607_b200 import _capi as capi
    from paper_1812_07607_b200 import patchdb

    cfg = JOINS[which]
    dev_index = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    lib = capi.lib()
    cos = cfg["kind"] == "cos"
    dt = torch.int16 if cos else torch.float32

    # ---- data ----------------------------------------------------------------
    # Cross joins (config 3): L is row-sharded -- rank k holds only its
    # contiguous rows [l0, l1) and joins them against all of R as a plain
    # cross join (so its band plan covers only its own L rows), and R is
    # generated on rank 0 and broadcast once over NCCL.  The seeded generator
    # is deterministic, so each rank slices its L rows from its own copy (a
    # loader would read just that range).  Self-joins (configs 1, 4, 5): rank
    # 0 generates X and broadcasts it; every rank scans its boustrophedon
    # share of the 128-row blocks (pdb_join_opts.shard_*).
    planted = None
    cross_shard = not cfg["self_join"] and world > 1
    if rank == 0 or cross_shard:
        if which == "c3":
            from paper_1812_07607_b200 import workloads
            Lh, Rh, pl_, pr_ = workloads.config3()
            planted = (pl_, pr_)
        else:
            Lh, Rh = _gen(which)
        shape_L = list(Lh.shape)
        shape_R = list(Rh.shape) if Rh is not None else [0, 0]
    else:
        Lh = Rh = None
        shape_L = shape_R = None
    if world > 1:
        box = [shape_L, shape_R]
        dist.broadcast_object_list(box, src=0)
        shape_L, shape_R = box
    nL_all, d = shape_L
    l0, l1 = (nL_all * rank // world, nL_all * (rank + 1) // world) if cross_shard else (0, nL_all)
    if cross_shard:
        Ld = torch.from_numpy(np.ascontiguousarray(Lh[l0:l1])).to(dev)
    else:
        Ld = (torch.from_numpy(Lh.view(np.int16) if cos else Lh).to(dev) if rank == 0
              else torch.empty(shape_L, dtype=dt, device=dev))
    Rd = None
    if shape_R[0]:
        Rd = torch.from_numpy(Rh).to(dev) if rank == 0 else torch.empty(shape_R, dtype=dt,
                                                                         device=dev)
    setup_ms = 0.0
    if world > 1:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if not cross_shard:
            dist.broadcast(Ld, src=0)
        if Rd is not None:
            dist.broadcast(Rd, src=0)  # the right relation, once
        e1.record()
        torch.cuda.synchronize()
        setup_ms = e0.elapsed_time(e1)
    nL = l1 - l0  # this rank's L rows
    nR = shape_R[0] if Rd is not None else nL
    cand = nL_all * (nL_all - 1) / 2 if cfg["self_join"] else float(nL_all) * nR

    stream = torch.cuda.current_stream(dev)
    sptr = C.c_void_p(stream.cuda_stream)
    pairs = patchdb.DevicePairs()

    def opts(phases):
        o = capi.JoinOpts()
        o.flags = ((capi.PDB_JOIN_SELF if cfg["self_join"] else 0) |
                   (capi.PDB_JOIN_PHASE_TIMES if phases else 0))
        # (a row-sharded cross join is a plain join of this rank's L rows)
        o.shard_index, o.shard_count = (0, 1) if cross_shard else (rank, world)
        o.stream = sptr
        return o

    o_plain, o_ph = opts(False), opts(True)
    Rp = Rd.data_ptr() if Rd is not None else Ld.data_ptr()
    fn = lib.pdb_cosine_join_bf16_dev if cos else lib.pdb_sim_join_dev

    def join(phases):
        rc = fn(Ld.data_ptr(), nL, Rp, nR, d, float(cfg["tau"]),
                C.byref(o_ph if phases else o_plain), C.byref(pairs._p), C.byref(pairs.stats))
        assert rc == 0, capi.last_error()

    # L2 flush by a 256 MB read (clean lines: no write-back inside the step)
    flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times, screen, recheck, prep, tiles, launches = [], [], [], [], [], 0

    def step(timed, phases=False):
        nonlocal launches
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        flush.amax()  # queued first: the host enqueues the join while it runs
        ev0.record(stream)
        join(phases)
        ev1.record(stream)
        torch.cuda.synchronize()
        if timed and not phases:
            times.append(ev0.elapsed_time(ev1))
            launches += pairs.stats.launches
        if timed and phases:
            st = pairs.stats
            screen.append(st.screen_ms)
            recheck.append(st.recheck_ms)
            prep.append(st.prep_ms)
            tiles.append(st.tiles)

    for _ in range(args.warmup):
        step(False)
    sampler = clock_sampler(dev_index)
    sampler.__enter__()
    for _ in range(args.steps):
        step(True)
    for _ in range(args.steps):
        step(True, phases=True)

    def maxred(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = maxred(statistics.mean(times))
    ms_screen = maxred(statistics.mean(screen))
    ms_recheck = maxred(statistics.mean(recheck))
    ms_prep = maxred(statistics.mean(prep))
    tot = torch.tensor([pairs.count, pairs.stats.candidates], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    n_pairs, n_cand = int(tot[0]), int(tot[1])
    # screened 128x256 tiles (the band plan skips separated ones), max over ranks
    tiles_rank = int(maxred(statistics.mean(tiles))) if tiles else 0
    nbl_, nt_ = -(-nL // 128), -(-nR // 256)
    tiles_dense = (sum(nt_ - rb // 2 for rb in range(nbl_)) if cfg["self_join"] else nbl_ * nt_)
    pairs.free()

    # ---- e2e: pinned host relations -> host C-ABI call -> host pairs --------
    e2e_steps = 1 if which == "c5" else max(1, min(args.steps, 3))
    Lhost = torch.empty(tuple(Ld.shape), dtype=dt, pin_memory=True)
    Lhost.copy_(Ld)
    Rhost = None
    if Rd is not None:
        Rhost = torch.empty(tuple(shape_R), dtype=dt, pin_memory=True)
        Rhost.copy_(Rd)
    hfn = lib.pdb_cosine_join_bf16 if cos else lib.pdb_sim_join
    e2e_t = []
    d2h = 0
    last_pairs = None
    for k in range(e2e_steps + 1):
        if world > 1:
            dist.barrier()
        o = opts(False)
        o.stream = None
        pr = capi.Pairs()
        t0 = time.perf_counter()
        rc = hfn(Lhost.data_ptr(), nL, Rhost.data_ptr() if Rhost is not None else Lhost.data_ptr(),
                 nR, d, float(cfg["tau"]), C.byref(o), C.byref(pr))
        t1 = time.perf_counter()
        assert rc == 0, capi.last_error()
        d2h = int(pr.count) * 12
        if which == "c3" and rank == 0 and k == e2e_steps:
            npr = int(pr.count)
            last_pairs = (np.ctypeslib.as_array(pr.left, (max(npr, 1),))[:npr].copy(),
                          np.ctypeslib.as_array(pr.right, (max(npr, 1),))[:npr].copy())
        lib.pdb_pairs_free(C.byref(pr))
        if k > 0:  # first call warms the pool / host allocator
            e2e_t.append(t1 - t0)
    sampler.__exit__()
    e2e_s = maxred(statistics.mean(e2e_t))
    h2d = Lhost.numel() * Lhost.element_size() + (Rhost.numel() * Rhost.element_size()
                                                  if Rhost is not None else 0)

    # ---- the dense screen (no band plan) on the same join: the tensor-pipe
    # roofline of K2 with nothing pruned --------------------------------------
    dense_rec = None
    if dense and not cos:
        o_d = opts(True)
        o_d.flags |= capi.PDB_JOIN_DENSE
        dp = patchdb.DevicePairs()
        dms, dscreen, dtiles = [], [], 0
        for k in range(3):
            torch.cuda.synchronize()
            flush.amax()
            ev0.record(stream)
            rc = fn(Ld.data_ptr(), nL, Rp, nR, d, float(cfg["tau"]), C.byref(o_d), C.byref(dp._p),
                    C.byref(dp.stats))
            ev1.record(stream)
            torch.cuda.synchronize()
            assert rc == 0, capi.last_error()
            if k:
                dms.append(ev0.elapsed_time(ev1))
                dscreen.append(dp.stats.screen_ms)
                dtiles = int(dp.stats.tiles)
        dense_pairs = dp.count
        dp.free()
        bpk = peaks.get("bf16_tflops") or 1590.0
        dflops = dtiles * 128 * 256 * 2 * d
        dtf = dflops / (statistics.mean(dscreen) * 1e-3) / 1e12
        dense_rec = {"ms_per_step": statistics.mean(dms), "screen_ms": statistics.mean(dscreen),
                     "gpairs_per_s": cand / (statistics.mean(dms) * 1e-3) / 1e9 / 1,
                     "tiles_screened": dtiles, "pairs": int(dense_pairs),
                     "roofline": {"kernel": "k_screen, dense plan (every 128x256 tile)",
                                  "bound": "tensor", "achieved": dtf, "peak": bpk,
                                  "unit": "TFLOP/s", "frac": dtf / bpk,
                                  "algorithmic": f"{dtiles} tiles x 128 x 256 x 2*{d} flop"}}

    # ---- config 4 as BASELINE.json states it (no planted near-duplicates):
    # independent ReLU'd projections sit near cosine ~0.3, so the join is
    # empty; the line's main workload plants 0.5 % near-duplicates so that
    # its parity check has pairs to check ---------------------------------------
    as_stated = None
    if which == "c4" and world == 1:
        from paper_1812_07607_b200 import workloads
        Xs = workloads.config4(device="cuda", plant_frac=0.0).view(torch.int16)
        sp = patchdb.DevicePairs()
        o_s = opts(False)
        st_ms = []
        for k in range(args.warmup + max(1, min(args.steps, 5))):
            torch.cuda.synchronize()
            flush.amax()
            ev0.record(stream)
            rc = lib.pdb_cosine_join_bf16_dev(Xs.data_ptr(), Xs.shape[0], Xs.data_ptr(), Xs.shape[0],
                                              Xs.shape[1], float(cfg["tau"]), C.byref(o_s),
                                              C.byref(sp._p), C.byref(sp.stats))
            ev1.record(stream)
            torch.cuda.synchronize()
            assert rc == 0, capi.last_error()
            if k >= args.warmup:
                st_ms.append(ev0.elapsed_time(ev1))
        n4 = Xs.shape[0]
        as_stated = {"workload": "config4 exactly as BASELINE.json states it (no planted pairs)",
                     "pairs": int(sp.count), "candidates": int(sp.stats.candidates),
                     "ms_per_step": statistics.mean(st_ms),
                     "value": n4 * (n4 - 1) / 2 / (statistics.mean(st_ms) * 1e-3) / 1e9,
                     "unit": "Gpairs/s"}
        sp.free()
        del Xs

    cpu = None
    checked = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            Lc = Lhost.numpy().view(np.uint16) if cos else Lhost.numpy()
            Rc = None if Rhost is None else Rhost.numpy()
            if which == "c3" and planted is not None and last_pairs is not None:
                cpu, checked = _verify_c3(Lc, Rc, planted, last_pairs[0], last_pairs[1],
                                          os.cpu_count() or 1)
            else:
                cpu = _cpu_baseline(which, Lc, Rc, cfg, os.cpu_count() or 1)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "Gpairs/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        bpeak = peaks.get("bf16_tflops") or 1590.0
        # one rank's screened tiles x 2d flop per pair (cosine: the dense plan)
        flops = (tiles_rank * 128 * 256 * 2 * d) if tiles_rank else cand * 2 * d / world
        screen_tf = flops / (ms_screen * 1e-3) / 1e12
        hbm = peaks.get("hbm_gbs", 6650.0)
        out_gbs = n_pairs * 12 / world / (ms_recheck * 1e-3) / 1e9 if ms_recheck > 0 else None
        line = {
            "metric": metric, "value": cand / (ms * 1e-3) / 1e9, "unit": "Gpairs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": ("fp16 screen / f64 exact" if int(pairs.stats.screen_format) == 2 else
                      "bf16 screen / f64 exact") if not cos else "bf16 screen / f64 exact (cosine)",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "nL": nL_all, "nL_per_rank": nL, "nR": nR, "d": d,
                       "threshold": cfg["tau"], "candidate_pairs": cand,
                       "l2": "flushed (256 MB read) before each step",
                       "parallelism": ("single GPU" if world == 1 else
                                       f"L rows sharded contiguously x{world} (each rank's band plan "
                                       f"covers its own L rows), R broadcast once over NCCL"
                                       if cross_shard else
                                       f"L row blocks boustrophedon x{world}, X broadcast once")},
            "pairs": n_pairs, "candidates": n_cand,
            "phase_ms": {"prep": ms_prep, "screen": ms_screen, "recheck": ms_recheck},
            "setup_ms": {"broadcast": setup_ms},
            "roofline": {"kernel": "k_screen (K2, tcgen05 kind::f16 on %s screen copies)"
                                   % {0: "tf32", 1: "bf16", 2: "fp16", 3: "bf16 (cosine)"}.get(
                                       int(pairs.stats.screen_format), "bf16"),
                         "bound": "tensor", "achieved": screen_tf, "peak": bpeak,
                         "unit": "TFLOP/s", "frac": screen_tf / bpeak,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)",
                         "algorithmic": f"{tiles_rank} screened 128x256 tiles per rank (of "
                                        f"{tiles_dense} dense) x 2*{d} flop per pair",
                         "tiles_screened": tiles_rank, "tiles_dense": tiles_dense,
                         "ms": ms_screen, "traffic": None},
            "roofline_output": {"kernel": "k_recheck (K3)", "bound": "hbm",
                                "achieved": out_gbs, "peak": hbm, "unit": "GB/s",
                                "frac": out_gbs / hbm if out_gbs else None,
                                "algorithmic": "12 B per emitted pair"},
            "cpu_baseline": cpu,
            "e2e": {"value": cand / e2e_s / 1e9, "unit": "Gpairs/s",
                    "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_s * 1e3,
                    "api": ("pdb_cosine_join_bf16" if cos else "pdb_sim_join") +
                           " (pinned host relations -> host pairs)"},
            "gpu_launches": launches,
            "clocks": sampler.summary(),
        }
        # the band plan screens only tiles whose projected boxes lie within
        # tau: the same join as if every tile were screened at this rate
        line["dense_equivalent"] = {
            "achieved": cand * 2 * d / world / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "note": "candidate pairs x 2d flop / step time: the dense GEMM work the exact band "
                    "plan avoids, credited as if done (not a tensor-pipe rate)"}
        if dense_rec is not None:
            line["dense_screen"] = dense_rec
        if checked is not None:
            line["checked"] = checked
        if as_stated is not None:
            line["as_stated"] = as_stated
        return line
    return None


# ---------------------------------------------------------------------------
# Dedup line (--workload dedup): the paper's near-duplicate grouping
# (run_dedup semantics) of the config-2 tile histograms.  One step = one
# pdb_dedup_dev over the 64,000 device-resident features; value = items/s.

def run_dedup_ours(args, rank, world, local_rank, metric, peaks, clock_sampler):
    import torch

    from paper_1812_07607_b200 import _capi as capi
    from paper_1812_07607_b200 import patchdb

    cfg = JOINS["dedup"]
    if rank != 0:  # a global sequential scan: one GPU runs it ("replicas only")
        return 0
    dev = torch.device("cuda", local_rank % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    Xh, _ = _gen("dedup")
    X = torch.from_numpy(Xh).to(dev)
    n, d = X.shape
    stream = torch.cuda.current_stream(dev)
    flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    nr = 0
    for k in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        flush.amax()  # (a read: clean L2 lines)
        ev0.record(stream)
        rep_of, nr = patchdb.dedup_device(X, cfg["tau"], stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        if k >= args.warmup:
            times.append(ev0.elapsed_time(ev1))
    sampler = clock_sampler(dev.index)
    sampler.__enter__()
    e2e = []
    for k in range(max(1, min(args.steps, 3)) + 1):
        t0 = time.perf_counter()
        g = patchdb.dedup(Xh, cfg["tau"])
        t1 = time.perf_counter()
        if k:
            e2e.append(t1 - t0)
    sampler.__exit__()
    ms = statistics.mean(times)
    e2e_s = statistics.mean(e2e)
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = _cpu_baseline("dedup", Xh, None, cfg, 1)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "items/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    # roofline: the tau-graph's screen dominates -- credit the flops of the
    # tiles it screens (the self-join's stats) over the whole dedup step (a
    # lower bound on the screen's rate)
    probe = patchdb.sim_join_device(X, None, cfg["tau"], self_join=True)
    tiles = int(probe.stats.tiles)
    probe.free()
    flops = tiles * 128 * 256 * 2 * d
    tf = flops / (ms * 1e-3) / 1e12
    bpeak = peaks.get("bf16_tflops") or 1590.0
    print(json.dumps({
        "metric": metric, "value": n / (ms * 1e-3), "unit": "items/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "replicas only", "vs_baseline": None, "dtype": "bf16 screen / f64 exact",
        "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": int(n), "d": int(d), "tau": cfg["tau"],
                   "l2": "flushed (256 MB read) before each step"},
        "reps": int(nr), "groups_with_members": int(sum(1 for m in g.members if len(m) > 1)),
        "roofline": {"kernel": "whole dedup step vs the tau-graph screen's algorithmic flops "
                               "(k_screen dominates)", "bound": "tensor", "achieved": tf,
                     "peak": bpeak, "unit": "TFLOP/s", "frac": tf / bpeak,
                     "algorithmic": f"{tiles} screened 128x256 tiles x 2*{d} flop per pair",
                     "ms": ms,
                     "traffic": None},
        "cpu_baseline": cpu,
        "e2e": {"value": n / e2e_s, "unit": "items/s", "h2d_bytes_per_step": int(Xh.nbytes),
                "d2h_bytes_per_step": int(n * 8), "ms_per_step": e2e_s * 1e3,
                "api": "pdb_dedup (host features -> host rep_of)"},
        "gpu_launches": None,
        "clocks": sampler.summary(),
    }))
    return 0


def run_dedup_reference(args, rank, world, metric):
    if rank != 0:
        return 0
    cfg = JOINS["dedup"]
    from oracle import oracle
    from paper_1812_07607_b200 import workloads
    fr, _ = workloads.frames(1000, 480, 640, seed=2)
    X = oracle.featurize_tiles(fr, 60, 80, 4, 1)
    vals, base = [], None
    for k in range(args.warmup + args.steps):
        base = _cpu_baseline("dedup", X, None, cfg, 1)
        if k >= args.warmup:
            vals.append(base["value"])
    v = statistics.mean(vals)
    base["value"] = v
    print(json.dumps({
        "impl": "reference", "metric": metric, "value": v, "unit": "items/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": X.shape[0] / v * 1e3,
        "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": int(X.shape[0])},
        "cpu_baseline": base,
        "e2e": {"value": v, "unit": "items/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0

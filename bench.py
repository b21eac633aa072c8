#!/usr/bin/env python
"""Benchmark of the hot path on BASELINE.json's configs[1] workload (config 2):

    1000 synthetic 480x640 uint8 frames -> 8x8 grid of 60x80 tiles (64,000)
    -> 4x4x4 joint colour histograms (64-d fp32, K1)
    -> L2 self-join, eps = 0.05, all (i<j, dist) pairs (K2 screen + K3 re-check)

One step = one pass of that pipeline over the 1000 frames.  ``value`` is
frames/s with the frames already resident in HBM (device-timed with CUDA
events, L2 flushed between steps); ``e2e`` is the same metric through the
public C-ABI call pdb_featurize_join with pinned host frames in and host
pairs out, copies inside the timed region.  The join alone is reported in
Gpairs/s (N(N-1)/2 candidate pairs per step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c5]

--workload c1/c3/c4/c5 prints the join-only line of that BASELINE config
instead (bench_join.py); the default line is config 2.

N > 1 runs under torchrun, one process per GPU: each rank featurizes its
frame shard, the 64,000 features are all-gathered over NCCL (16 MB), and
each rank joins the 128-row blocks b = rank (mod N) of the features against
all of them (strong scaling: the 1000-frame workload is fixed).
``--impl reference`` times the reference's own CPU implementation
(oracle/_ref, the unmodified proj/ sources) on the host cores instead: every
timed step is the full config-2 step (all 1000 frames, the ball-tree join
of all 64,000 features), on all host cores or --ref-threads N.

The default line also carries ``config3``: the north-star join
(1,048,576 x 1,048,576 x 128, tau 0.02) measured in the same run -- device
and e2e Gpairs/s, the screen's tensor roofline on the tiles it screens, a
dense-screen pass of the same join, and the reference's own probe output on
sampled rows compared with the GPU's (``checked``).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(frames=1000, H=480, W=640, tile_h=60, tile_w=80, bins=4, mode="joint", tau=0.05,
           seed=2)
METRIC = "similarity-join Gpairs/s + featurization frames/s, 1/2/4/8 B200 vs host-CPU ref"
WORKLOAD = "config2_featurize_join: 1000x480x640 u8 frames -> 64000 tiles 60x80 -> joint 4x4x4 hist (64-d) -> L2 self-join eps=0.05"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    tf32 = None
    try:
        tf32 = json.load(open(os.path.join(ROOT, "profiles", "peaks_tf32.json")))
    except Exception:
        pass
    return p, tf32


class ClockSampler:
    """Polls SM clock and throttle reasons through NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        return {"sm_mhz": int(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own implementation on the host cores.

def reference_step(frames: np.ndarray, feats: np.ndarray, threads: int, frames_n=None,
                   probe_rows=None):
    """One config-2 step of the reference itself (oracle/_ref, the unmodified
    proj/ sources), on `threads` host threads:

    * featurization: transform(generate(frames, tiles 80x60), color_histogram
      {B=4}) (src/etl.cpp:264-373) -- the reference's per-channel operator;
      it has no joint mode, whose binning cost is the same -- frames sharded
      over the threads;
    * the self-join of the 64,000 features: build_balltree over all of them
      plus balltree_within(0.05) for every probe row (run_sim_join's probe
      loop, src/query.cpp:516-526, over probe-row shards sharing the
      immutable tree).

    With frames_n / probe_rows set, only that many frames / probe rows run
    and the seconds are extrapolated linearly (the single-thread sample).
    Returns (featurize_s, join_s, info)."""
    from oracle import oracle
    if oracle.ref() is None:
        raise RuntimeError("oracle/_ref/libpdb_ref.so missing")
    fr = frames if frames_n is None else frames[:frames_n]
    t0 = time.perf_counter()
    oracle.ref_featurize_tiles(fr, CFG["tile_h"], CFG["tile_w"], CFG["bins"], threads=threads)
    t_feat = (time.perf_counter() - t0) * CFG["frames"] / fr.shape[0]
    n = feats.shape[0]
    rows = n if probe_rows is None else min(probe_rows, n)
    # a sample spreads its probe rows evenly over the relation
    sub = feats if rows == n else np.ascontiguousarray(feats[:: max(1, n // rows)][:rows])
    m, t_build, t_probe = _probe(sub, feats, threads)
    t_join = t_build + t_probe * n / rows
    return t_feat, t_join, {"frames": int(fr.shape[0]), "probe_rows": rows, "build_s": t_build,
                            "probe_s": t_probe, "matches": m}


def _probe(sub, feats, threads):
    from oracle import oracle
    import ctypes as C
    R = np.ascontiguousarray(feats, dtype=np.float32)
    L = np.ascontiguousarray(sub, dtype=np.float32)
    b, p = C.c_double(), C.c_double()
    # self_join=0: every probe row is matched against the whole tree, as the
    # reference's sim_join(X, X) does (the i < j view drops half afterwards)
    m = oracle.ref().ref_join_probe_timed(L.ctypes.data, L.shape[0], R.ctypes.data, R.shape[0],
                                          R.shape[1], CFG["tau"], 0, 0, L.shape[0], threads,
                                          C.byref(b), C.byref(p))
    return int(m), b.value, p.value


def _ref_inputs():
    from paper_1812_07607_b200 import workloads
    from oracle import oracle
    frames, _ = workloads.frames(CFG["frames"], CFG["H"], CFG["W"], seed=CFG["seed"])
    # the features the reference joins are the K1 output definition; compute
    # them with the restatement's bit-identical CPU code (no GPU in this arm)
    feats = oracle.featurize_tiles(frames, CFG["tile_h"], CFG["tile_w"], CFG["bins"], 1)
    return frames, feats


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    threads = args.ref_threads or os.cpu_count() or 1
    frames, feats = _ref_inputs()
    # Warm-up steps page the reference's code and the inputs in on a small
    # slice (1 frame, 64 probe rows); every TIMED step is the full workload:
    # all 1000 frames and all 64,000 probe rows, nothing extrapolated.
    for _ in range(args.warmup):
        reference_step(frames, feats, threads, frames_n=1, probe_rows=64)
    times, info = [], None
    for _ in range(args.steps):
        t_feat, t_join, info = reference_step(frames, feats, threads)
        times.append((t_feat, t_join))
    step_s = statistics.mean(a + b for a, b in times)
    join_s = statistics.mean(b for _, b in times)
    value = CFG["frames"] / step_s
    n = feats.shape[0]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8/f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "frames": CFG["frames"], "tiles": n, "d": 64,
                   "tau": CFG["tau"]},
        "join_gpairs_per_s": n * (n - 1) / 2 / join_s / 1e9,
        "phase_s": {"featurize": statistics.mean(a for a, _ in times), "join": join_s,
                    "join_build": info["build_s"], "join_probe": info["probe_s"]},
        "extrapolated": False,
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "reference",
                         "sample": f"the full step every timed step: reference transform(generate("
                                   f"tiles),color_histogram) of all {info['frames']} frames + "
                                   f"build_balltree({n}) and balltree_within for all "
                                   f"{info['probe_rows']} probe rows, {threads} threads"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# Our arm.

def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1812_07607_b200 import _capi as capi
    from paper_1812_07607_b200 import patchdb, workloads

    dev_index = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    lib = capi.lib()
    F, H, W, th, tw, B = (CFG[k] for k in ("frames", "H", "W", "tile_h", "tile_w", "bins"))
    tau = CFG["tau"]
    mode = capi.PDB_HIST_JOINT
    D = B ** 3
    tpf = (H // th) * (W // tw)
    f0, f1 = F * rank // world, F * (rank + 1) // world
    nf = f1 - f0
    n_tiles = F * tpf

    # pinned host frames of this rank's shard (the e2e input) + a device copy
    hbuf = lib.pdb_host_alloc(nf * H * W * 3)
    assert hbuf, "pinned allocation failed"
    host = np.ctypeslib.as_array(C.cast(hbuf, C.POINTER(C.c_uint8)), shape=(nf, H, W, 3))
    workloads.frames(nf, H, W, seed=CFG["seed"], first=f0, out=host)
    d_frames = torch.from_numpy(host).to(dev)
    feats = torch.empty((n_tiles, D), dtype=torch.float32, device=dev)
    my_feats = feats[f0 * tpf:f1 * tpf] if world == 1 else torch.empty((nf * tpf, D),
                                                                        dtype=torch.float32,
                                                                        device=dev)
    # L2 flush: a read of 256 MB (> the 126 MB L2) before each step.  A read
    # leaves clean lines: a written flush buffer would leave ~126 MB of dirty
    # lines whose write-back lands inside the next step's timed region.
    flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()

    def l2_flush():
        return flush.amax()
    stream = torch.cuda.current_stream(dev)
    sptr = C.c_void_p(stream.cuda_stream)
    pairs = patchdb.DevicePairs()
    opts = capi.JoinOpts()
    opts.flags = capi.PDB_JOIN_SELF
    opts.shard_index, opts.shard_count = rank, world
    opts.stream = sptr

    # Sharded steps fuse the feature all-gather into K1 (P2P stores into every
    # rank's matrix over NVLink, shard.PeerFeatures); PDB_P2P_FEATURES=0 keeps
    # the NCCL all-gather.
    p2p = None
    if world > 1 and os.environ.get("PDB_P2P_FEATURES", "1") != "0":
        from paper_1812_07607_b200 import shard
        try:
            p2p = shard.PeerFeatures(feats)
        except Exception as e:  # no IPC between these processes: NCCL path
            if rank == 0:
                print(f"P2P feature exchange unavailable ({e}); using all_gather", file=sys.stderr)
            p2p = None
    out_ptrs = None
    if p2p is not None:
        ptrs = p2p.ptrs(f0 * tpf * D)
        out_ptrs = (C.c_void_p * len(ptrs))(*ptrs)
    barrier_t = torch.zeros(1, dtype=torch.int32, device=dev)

    def featurize():
        if p2p is not None:
            rc = lib.pdb_featurize_tiles_dev_multi(d_frames.data_ptr(), nf, H, W, th, tw, B, mode,
                                                   out_ptrs, len(out_ptrs), sptr)
        else:
            rc = lib.pdb_featurize_tiles_dev(d_frames.data_ptr(), nf, H, W, th, tw, B, mode,
                                             my_feats.data_ptr(), sptr)
        assert rc == 0, capi.last_error()

    def gather():
        if world > 1 and p2p is not None:
            # every rank's K1 has stored into our matrix once all have passed
            # this point (K1 ends with a system-scope fence)
            if dist.get_backend() == "nccl":
                dist.all_reduce(barrier_t)
            else:
                torch.cuda.current_stream(dev).synchronize()
                dist.barrier()
        elif world > 1:
            if dist.get_backend() == "nccl":
                dist.all_gather_into_tensor(feats, my_feats)
            else:  # gloo (multi-rank smoke on one GPU): list all-gather
                parts = list(feats.split(my_feats.shape[0]))
                dist.all_gather(parts, my_feats)
                for k, part in enumerate(parts):
                    feats[k * my_feats.shape[0]:(k + 1) * my_feats.shape[0]].copy_(part)

    opts_ph = capi.JoinOpts()
    opts_ph.flags = capi.PDB_JOIN_SELF | capi.PDB_JOIN_PHASE_TIMES
    opts_ph.shard_index, opts_ph.shard_count = rank, world
    opts_ph.stream = sptr

    def join(phases=False):
        rc = lib.pdb_sim_join_dev(feats.data_ptr(), n_tiles, feats.data_ptr(), n_tiles, D, tau,
                                  C.byref(opts_ph if phases else opts), C.byref(pairs._p),
                                  C.byref(pairs.stats))
        assert rc == 0, capi.last_error()

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    rec = {"step": [], "feat": [], "gather": [], "join": [], "screen": [], "recheck": [], "tiles": [],
           "prep": []}
    launches = 0

    # one GPU: the step is one pdb_featurize_join_dev call (the band plan's
    # directions computed beside K1); sharded: featurize, exchange, join
    use_fused = world == 1 and not args.no_fused

    def fused():
        rc = lib.pdb_featurize_join_dev(d_frames.data_ptr(), nf, H, W, th, tw, B, mode, tau,
                                        C.byref(opts), feats.data_ptr(), C.byref(pairs._p),
                                        C.byref(pairs.stats))
        assert rc == 0, capi.last_error()

    def step(timed: bool, phases: bool = False, split: bool = False):
        nonlocal launches
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # the L2 flush is queued first: while the device reads it, the host
        # enqueues the step, so ev[0]..ev[3] time the device work alone
        # (not the host's launch latency on an idle device)
        l2_flush()
        ev[0].record(stream)
        if use_fused and not (phases or split):
            fused()
        else:
            featurize()
            ev[1].record(stream)
            gather()
            ev[2].record(stream)
            join(phases)
        ev[3].record(stream)
        torch.cuda.synchronize()
        if timed and not (phases or split):
            rec["step"].append(ev[0].elapsed_time(ev[3]))
            launches += pairs.stats.launches + (0 if use_fused else 1)
        if timed and (split or (not phases and not use_fused)):
            # the featurize / join split (separate calls, no join phase events)
            rec["feat"].append(ev[0].elapsed_time(ev[1]))
            rec["gather"].append(ev[1].elapsed_time(ev[2]))
            rec["join"].append(ev[2].elapsed_time(ev[3]))
        if timed and phases:
            st = pairs.stats
            rec["screen"].append(st.screen_ms)
            rec["recheck"].append(st.recheck_ms)
            rec["prep"].append(st.prep_ms)
            rec["tiles"].append(st.tiles)

    for _ in range(args.warmup):
        step(False)
    # clocks are sampled across both timed regions (device steps and e2e)
    sampler = ClockSampler(dev_index)
    sampler.__enter__()
    for _ in range(args.steps):
        step(True)
    if use_fused:
        for _ in range(args.steps):
            step(True, split=True)
    # the per-phase split (roofline of the screen kernel) comes from separate
    # steps with CUDA events between the join's phases; those events break
    # the programmatic-dependent-launch chain, so they stay out of `value`
    for _ in range(args.steps):
        step(True, phases=True)

    def maxred(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_step = maxred(statistics.mean(rec["step"]))
    ms_feat = maxred(statistics.mean(rec["feat"]))
    ms_join = maxred(statistics.mean(rec["join"]))
    ms_screen = maxred(statistics.mean(rec["screen"]))
    ms_recheck = maxred(statistics.mean(rec["recheck"]))
    ms_gather = maxred(statistics.mean(rec["gather"]))
    ms_prep = maxred(statistics.mean(rec["prep"]))
    n_pairs_local = pairs.count
    tot = torch.tensor([n_pairs_local, pairs.stats.candidates], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    n_pairs, n_cand = int(tot[0]), int(tot[1])

    # ---- e2e: host pinned frames -> public API -> host pairs -----------------
    e2e_times = []
    h2d = nf * H * W * 3
    d2h = 0
    for k in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            o = capi.JoinOpts()
            pr = capi.Pairs()
            rc = lib.pdb_featurize_join(hbuf, nf, H, W, th, tw, B, mode, tau, C.byref(o), None,
                                        C.byref(pr))
            assert rc == 0, capi.last_error()
            npairs = pr.count
            lib.pdb_pairs_free(C.byref(pr))
        else:
            d_frames.copy_(torch.from_numpy(host), non_blocking=True)
            featurize()
            gather()
            join()
            l_, r_, d_ = pairs.to_torch(dev, copy=False)
            hl = torch.empty(l_.shape, dtype=torch.int32, pin_memory=True)
            hr = torch.empty(r_.shape, dtype=torch.int32, pin_memory=True)
            hd = torch.empty(d_.shape, dtype=torch.float32, pin_memory=True)
            hl.copy_(l_)
            hr.copy_(r_)
            hd.copy_(d_)
            torch.cuda.synchronize()
            npairs = pairs.count
        t1 = time.perf_counter()
        d2h = npairs * 12
        if k >= args.warmup:
            e2e_times.append(t1 - t0)
    sampler.__exit__()
    e2e_s = maxred(statistics.mean(e2e_times))
    # the e2e path's own roofline: a plain pinned-host -> device copy of the
    # same bytes (PCIe), best of 3
    hx = torch.from_numpy(host)
    h2d_best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        d_frames.copy_(hx, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        h2d_best = t if h2d_best is None else min(h2d_best, t)
    h2d_gbs = maxred(h2d / h2d_best / 1e9)
    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            fh = feats.cpu().numpy()
            # the full step once on all host cores, nothing extrapolated ...
            t_feat, t_join, info = reference_step(host, fh, threads)
            v = F / (t_feat + t_join)
            cpu = {"value": v, "unit": "frames/s", "cores": threads, "kind": "reference",
                   "sample": f"the full step once: reference (oracle/_ref) featurization of all "
                             f"{info['frames']} frames (per-channel B=4 operator) + "
                             f"build_balltree({fh.shape[0]}) and balltree_within for all "
                             f"{info['probe_rows']} probe rows, {threads} threads",
                   "featurize_s": t_feat, "join_s": t_join, "extrapolated": False}
            # ... and single-threaded as the reference ships, on a
            # bounded sample: 32 frames + 1024 evenly spread probe rows
            t1f, t1j, i1 = reference_step(host, fh, 1, frames_n=32, probe_rows=1024)
            cpu["single_thread"] = {
                "value": F / (t1f + t1j), "unit": "frames/s", "cores": 1, "kind": "reference",
                "sample": f"{i1['frames']} frames + build_balltree({fh.shape[0]}) and "
                          f"{i1['probe_rows']} evenly spread probe rows on 1 thread, "
                          f"extrapolated linearly to 1000 frames / {fh.shape[0]} probe rows",
                "featurize_s": t1f, "join_s": t1j, "extrapolated": True}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "frames/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # ---- the north-star join (config 3), measured in the same run ----------
    c3 = None
    if not args.no_config3:
        import bench_join
        c3_args = argparse.Namespace(**vars(args))
        c3_args.steps = min(args.steps, 10)
        c3 = bench_join.measure(c3_args, rank, world, local_rank, "c3", METRIC, peaks()[0],
                                ClockSampler, dense=True)

    if rank == 0:
        mp, _ = peaks()
        pairs_cand = n_tiles * (n_tiles - 1) / 2
        hbm = mp.get("hbm_gbs", 6650.0)
        feat_bytes = F * (H * W * 3 + tpf * D * 4) / world
        feat_gbs = feat_bytes / (ms_feat * 1e-3) / 1e9
        # the band plan screens only the 128x256 tiles whose projected boxes
        # lie within tau; the roofline credits the tiles actually screened
        nt_ = -(-n_tiles // 256)
        tiles_dense = sum(nt_ - rb // 2 for rb in range(-(-n_tiles // 128)))
        tiles_screened = int(statistics.mean(rec["tiles"])) if rec["tiles"] else tiles_dense
        flops = tiles_screened * 128 * 256 * 2 * D / world
        screen_tflops = flops / (ms_screen * 1e-3) / 1e12
        # the screen runs tcgen05 kind::f16 on bf16 copies: its roofline is the
        # measured dense bf16 peak (MEASURED_PEAKS.json, burst: a kernel timed alone)
        bpeak = mp.get("bf16_tflops")
        bsrc = "MEASURED_PEAKS.json bf16_tflops (burst)"
        if not bpeak:
            bpeak, bsrc = 1590.0, "B200_PROFILING.md fallback 1.59 PFLOP/s"
        traffic = None
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        except Exception:
            pass
        rl_screen = {"kernel": "k_screen (K2, tcgen05 kind::f16 on bf16 screen copies)",
                     "bound": "tensor", "achieved": screen_tflops, "peak": bpeak,
                     "unit": "TFLOP/s", "frac": screen_tflops / bpeak, "peak_source": bsrc,
                     "frac_of_sustained_bf16": screen_tflops / mp.get("bf16_tflops_sustained", bpeak),
                     "algorithmic": f"{tiles_screened} screened 128x256 tiles (of {tiles_dense} in "
                                    f"the triangle) x 2*{D} flop per pair",
                     "tiles_screened": tiles_screened, "tiles_dense": tiles_dense,
                     "ms": ms_screen,
                     "traffic": (traffic or {}).get("k_screen")}
        rl_feat = {"kernel": "k_hist_joint_rows8 (K1, TMA-fed, 8-bit lane counters)", "bound": "hbm", "achieved": feat_gbs,
                   "peak": hbm, "unit": "GB/s", "frac": feat_gbs / hbm,
                   "algorithmic": "937,984 B/frame (921,600 read + 64 x 64 x 4 written)",
                   "ms": ms_feat, "traffic": (traffic or {}).get("k_hist_joint_rows8")}
        dominant = rl_screen if ms_screen >= ms_feat else rl_feat
        line = {
            "metric": METRIC, "value": F / (ms_step * 1e-3), "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8 hist / bf16 screen / f64 exact", "data": "synthetic",
            "config": {"workload": WORKLOAD, "frames": F, "tiles": n_tiles, "d": D, "tau": tau,
                       "candidate_pairs": pairs_cand, "l2": "flushed (256 MB read) before each step",
                       "parallelism": f"frames sharded x{world}, "
                       + ("features P2P-stored by K1 into every rank's matrix (fused all-gather)"
                          if p2p is not None else "features all-gathered")
                       + f", join row-blocks cyclic x{world}",
                       "step_api": ("pdb_featurize_join_dev (the band plan's directions computed "
                                    "beside K1); phase_ms from separate featurize / join calls"
                                    if use_fused else
                                    "pdb_featurize_tiles_dev + exchange + pdb_sim_join_dev")},
            "join_gpairs_per_s": pairs_cand / (ms_join * 1e-3) / 1e9,
            "featurize_frames_per_s": F / (ms_feat * 1e-3),
            "phase_ms": {"featurize": ms_feat, "gather": ms_gather,
                         "join": ms_join, "join_prep": ms_prep,
                         "join_screen": ms_screen, "join_recheck": ms_recheck},
            "pairs": n_pairs, "candidates": n_cand,
            "roofline": dominant, "roofline_all": [rl_feat, rl_screen],
            "cpu_baseline": cpu,
            "e2e": {"value": F / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": h2d * world,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                    "roofline": {"bound": "pcie_h2d", "achieved": h2d / e2e_s / 1e9,
                                 "peak": h2d_gbs, "unit": "GB/s",
                                 "frac": (h2d / e2e_s / 1e9) / h2d_gbs,
                                 "peak_source": "pinned host -> device copy of the same frames, "
                                                "measured in this run (best of 3)"},
                    "api": "pdb_featurize_join (pinned host frames -> host pairs)" if world == 1
                           else "featurize_tiles_dev + all_gather + pdb_sim_join_dev + D2H"},
            "gpu_launches": launches,
            "clocks": sampler.summary(),
        }
        if c3 is not None:
            line["config3"] = c3
        print(json.dumps(line))
    pairs.free()
    lib.pdb_host_free(hbuf)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused", action="store_true",
                    help="time the config-2 step as separate featurize and join calls instead of "
                         "pdb_featurize_join_dev")
    ap.add_argument("--no-config3", action="store_true",
                    help="skip the config-3 (1M x 1M x 128) sub-record of the default line")
    ap.add_argument("--ref-threads", type=int, default=0,
                    help="--impl reference: host threads (default: all cores; 1 = the "
                         "reference as shipped)")
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "dedup"],
                    help="c2 (default, the headline): featurize -> join pipeline; c1/c3/c4/c5: "
                         "the join-only configs of BASELINE.json (bench_join.py)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.workload != "c2":
        import bench_join
        if args.impl == "reference":
            if args.workload == "dedup":
                return bench_join.run_dedup_reference(args, rank, world, METRIC)
            return bench_join.run_reference(args, rank, world, args.workload, METRIC)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        dev_index = local_rank % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(dev_index)
        # PDB_DIST_BACKEND=gloo runs the multi-rank code path on fewer GPUs
        # than ranks (host collectives; kernels of different ranks never wait
        # on one another).  Real runs use NCCL, one process per GPU.
        backend = os.environ.get("PDB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    try:
        if args.workload != "c2":
            import bench_join
            if args.workload == "dedup":
                return bench_join.run_dedup_ours(args, rank, world, local_rank, METRIC,
                                                 peaks()[0], ClockSampler)
            return bench_join.run_ours(args, rank, world, local_rank, args.workload, METRIC,
                                       peaks()[0], ClockSampler)
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())

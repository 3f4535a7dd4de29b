"""Benchmark: ray-bounce segments/s into SH energy IRs (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

One step = one frame of the configured workload (default C5, BASELINE.json
configs[4], the largest config that fits one B200: 964,002-triangle city
grid, 256 sources x 2^20 paths, 100 bounces, 8 bands, order-3 SH histogram):
ef_trace (one persistent kernel over all paths of all sources, histogram
cleared by DMA first) followed by ef_analyze (per-band RT60/DRR/predelay/
loudness).  N > 1 (torchrun): strong scaling, the frame is fixed and rank g
traces rays [g*R/N, (g+1)*R/N) of every source (global Philox ray indices,
so the paths are those of the 1-GPU frame); the splats go straight to the
owning rank's histogram blocks inside the trace kernel (ef_trace_fused) or,
with --exchange nccl, one reduce-scatter per frame; each rank then analyses
its S/N sources.

Timing: CUDA events per step on the launching stream, L2 flushed (256 MiB
write) between steps outside the events, max over ranks.  ``e2e`` repeats
the steps through the public API with the source positions copied in from
pinned host memory and the frame's result -- the LowRateIR histograms and
direct blocks of the rank's sources (what trace_frame returns)
and the reverb parameters per source and band -- copied back to pinned host
memory, all inside the timed region.  ``--impl reference`` times the CPU oracle
port of the reference algorithm (oracle/efo.c, every host core) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic work per segment of the REFERENCE algorithm (tools/measure_work.py,
# DESIGN.md section 5): nodes visited / triangles tested by bvh.py:130-160
# (C1: all-pairs over 12 triangles), listener-arrival fraction.
WORK = {
    "c1": dict(N_node=0.0, N_tri=12.0, P_arr=0.011300),
    "c2": dict(N_node=32.304, N_tri=5.334, P_arr=0.0),
    # subsampled (tools/measure_work.py c3 2048 8 / c5 1024 16)
    "c3": dict(N_node=74.351, N_tri=12.123, P_arr=0.001952),
    "c5": dict(N_node=66.946, N_tri=7.966, P_arr=0.0),
}


def b_seg(cfg, n_bands, nk):
    w = WORK[cfg]
    return 72 * w["N_tri"] + 32 * w["N_node"] + (28 + 8 * n_bands) + w["P_arr"] * 8 * n_bands * nk


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region:
    ONE `nvidia-smi -lms` process (the profiling recipe's clocks line),
    started before the region (first sample awaited) and stopped after, so
    no per-sample process launch competes with the timed launches."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"

    def __init__(self, index=0, period_ms=100):
        self.index = index
        self.period_ms = period_ms
        self.samples = []
        self._p = None
        self._t = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                        "--format=csv,noheader,nounits", f"-lms={self.period_ms}"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._p = None
            return self
        first = threading.Event()

        def reader():
            for line in self._p.stdout:
                try:
                    sm, smax, reasons = [x.strip() for x in line.split(",")]
                    self.samples.append((float(sm), float(smax), int(reasons, 16)))
                    first.set()
                except ValueError:
                    pass

        self._t = threading.Thread(target=reader, daemon=True)
        self._t.start()
        first.wait(5.0)
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}
        bits = 0
        for s in self.samples:
            bits |= s[2]
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": [v for k, v in names.items() if bits & k and k != 0x1],
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------- CPU arm
def cpu_oracle_rate(w, rays_per_source, threads, min_seconds=0.0):
    """CPU port of the reference algorithm (oracle/efo.c, reference BVH and
    traversal, the pinned bounce loop) on `threads` host threads: each thread
    traces a contiguous ray shard of every source; whole frames (frame index
    0, 1, ...) repeat until `min_seconds` elapsed.  Returns (seg/s, segs, s,
    frames)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    os_ = O.OracleScene.from_arrays(w.arrays())
    bin_len = w.speed_of_sound * w.bin_s
    shards = []
    per = max(1, rays_per_source // threads)
    for s in range(len(w.sources)):
        for r0 in range(0, rays_per_source, per):
            shards.append((s, r0, min(per, rays_per_source - r0)))

    def run(job):
        s, r0, n, frame = job
        r = O.trace(os_, src_key=s, src_pos=w.sources[s], listener=w.listener, radius=w.radius,
                    seed=w.seed, frame=frame, order=w.order, n_bins=w.n_bins, bin_len=bin_len,
                    max_bounces=w.max_bounces, e0=1.0, ray0=r0, n_rays=n)
        return r.stats["segments"]

    segs, frames = 0, 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        while True:
            segs += sum(ex.map(run, [j + (frames,) for j in shards]))
            frames += 1
            if time.perf_counter() - t0 >= min_seconds:
                break
    dt = time.perf_counter() - t0
    return segs / dt, segs, dt, frames


def run_reference(args, w, metric, unit):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    rays = max(1, int(w.n_rays * args.cpu_fraction))
    for _ in range(min(args.warmup, 1)):
        cpu_oracle_rate(w, max(1, rays // 16), cores)
    rates, secs = [], []
    for _ in range(args.steps):
        r, segs, dt, _ = cpu_oracle_rate(w, rays, cores)
        rates.append(r)
        secs.append(dt)
    value = float(np.median(rates))
    sample = f"rays [0,{rays}) of each of the {len(w.sources)} sources of {w.name} per step"
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit,
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.median(secs)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, w, world),
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(args, w, world, exchange=None):
    exchange = exchange or args.exchange
    return {"workload": f"{w.name} (BASELINE.json configs[{ {'c1': 0, 'c2': 1, 'c3': 2, 'c5': 4}[args.config] }])",
            "triangles": int(w.n_tri), "sources": int(len(w.sources)),
            "rays_per_source": int(w.n_rays), "rays_per_source_per_rank": int(w.n_rays // world),
            "max_bounces": int(w.max_bounces),
            "sh_order": int(w.order), "bands": int(w.n_bands), "bins": int(w.n_bins),
            "parallelism": (f"each source's rays sharded x{world} (fixed frame), " + (
                "histograms reduce-scattered inside the trace kernel (ef_trace_fused, peer memory)"
                if exchange == "fused" else "NCCL reduce-scatter of histograms (ef_nccl_reduce_hist)")) if world > 1
            else "single GPU", "l2": "flushed between steps (256 MiB write)"}


# ----------------------------------------------------------------- GPU arm
def run_gpu(args, w, metric, unit):
    import torch
    import torch.distributed as dist

    from paper_1803_00430_b200 import _lib
    from paper_1803_00430_b200.analysis import Analyzer
    from paper_1803_00430_b200.propagation import FrameTracer, TraceConfig
    from paper_1803_00430_b200.scene import scene_from_workload

    world, rank, local = dist_env()
    local = local % torch.cuda.device_count()   # gloo plumbing runs may share one GPU
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:   # plumbing checks with several ranks on one GPU (fused exchange only)
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    sc = scene_from_workload(w)
    S = len(w.sources)
    cfg = TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                      bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    tr = FrameTracer(sc, S, cfg)
    tr.set_sources(w.sources)
    if world > 1 and S % world:
        raise SystemExit("sources must divide by the number of ranks")
    S_own = S // world
    an = Analyzer(S_own, w.n_bins, sc.n_bands, w.order, w.bin_s)
    nk = cfg.n_coeffs
    fused = world > 1 and args.exchange == "fused"
    exchange_note = None
    if fused:
        from paper_1803_00430_b200.distributed import PeerHistograms, PeerUnavailable
        try:
            peers = PeerHistograms(S, w.n_bins, sc.n_bands, cfg.n_coeffs)
            st_all = torch.empty_like(tr.stats)
            su_all = torch.empty_like(tr.sum_t)
        except PeerUnavailable as e:   # every rank falls back together
            fused = False
            exchange_note = f"fused exchange unavailable ({e}); NCCL reduce-scatter used"
    if world > 1 and not fused:
        # unfused exchange through the C ABI (ef_nccl_reduce_hist) for the
        # histograms; the small per-source counters through torch's NCCL
        from paper_1803_00430_b200.distributed import NcclHistExchange
        nccl_ex = NcclHistExchange(world, rank, local)
        H_own = torch.empty((S_own,) + tuple(tr.H.shape[1:]), dtype=torch.float32, device=dev)
        D_own = torch.empty((S_own,) + tuple(tr.Dir.shape[1:]), dtype=torch.float32, device=dev)
        st_own = torch.empty((S_own, tr.stats.shape[1]), dtype=torch.int64, device=dev)
        su_own = torch.empty((S_own,), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # scene (nodes + triangle records) + frame outputs larger than the 126 MB L2
    big_inputs = (sc.device_info()["device_bytes"] + tr._outputs.numel()) > (160 << 20)
    stream = torch.cuda.current_stream()
    # strong scaling: the frame is fixed; rank g traces rays [g*R/N, (g+1)*R/N)
    # of every source (global Philox ray index, e0 normalised by R)
    if w.n_rays % world:
        raise SystemExit("rays per source must divide by the number of ranks")
    total_rays = w.n_rays
    n_rays = w.n_rays // world
    ray0 = rank * n_rays
    # C3: moving sources, temporal IR cache (accumulate_ir, tau_LR = 3 s) and
    # per-frame estimation on the cached IR
    dynamic = w.n_frames > 1 and w.source_velocity is not None
    if dynamic:
        from paper_1803_00430_b200.analysis import blend_into
        from paper_1803_00430_b200.propagation import TAU_LR
        pos_all = torch.tensor(np.stack([w.source_positions(f) for f in range(w.n_frames)]),
                               dtype=torch.float64, device=dev)
        alpha = 1.0 - float(np.exp(-w.frame_dt / TAU_LR))
        H_cache = torch.zeros((S_own,) + tuple(tr.H.shape[1:]), dtype=torch.float32, device=dev)
        D_cache = torch.zeros((S_own,) + tuple(tr.Dir.shape[1:]), dtype=torch.float32, device=dev)
    seg_total = torch.zeros((), dtype=torch.int64, device=dev)
    tail_total = torch.zeros((), dtype=torch.int64, device=dev)
    work_total = torch.zeros(3, dtype=torch.int64, device=dev)   # nodes, triangles, arrivals
    counter = [0]

    def step(kernel_events=None):
        f = counter[0] % max(w.n_frames, 1)
        counter[0] += 1
        if dynamic:
            tr.src_pos.copy_(pos_all[f])
        seq = counter[0]
        if kernel_events:
            kernel_events[0].record(stream)
        if fused:
            peers.begin_frame(seq)
            tr.trace_fused(w.listener, peers, frame=f, ray0=ray0, n_rays=n_rays, total_rays=total_rays,
                           slot=seq)
        else:
            tr.trace(w.listener, frame=f, ray0=ray0, n_rays=n_rays, total_rays=total_rays)
        if kernel_events:
            kernel_events[1].record(stream)
        if fused:
            # the histograms are complete once every rank's trace finished;
            # the 88-byte-per-source counters take one small all-reduce
            st_all.copy_(tr.stats)
            su_all.copy_(tr.sum_t)
            dist.all_reduce(st_all)
            dist.all_reduce(su_all)
            peers.end_frame()
            hs, ds = peers.block(seq)
            own = slice(rank * S_own, (rank + 1) * S_own)
            sts, sus = st_all[own], su_all[own]
        elif world > 1:
            nccl_ex.reduce_scatter(tr.H, H_own)
            nccl_ex.reduce_scatter(tr.Dir, D_own)
            dist.reduce_scatter_tensor(st_own, tr.stats)
            dist.reduce_scatter_tensor(su_own, tr.sum_t)
            hs, ds, sts, sus = H_own, D_own, st_own, su_own
        else:
            hs, ds, sts, sus = tr.H, tr.Dir, tr.stats, tr.sum_t
        if dynamic:
            blend_into(H_cache, hs, alpha)
            blend_into(D_cache, ds, alpha)
            hs, ds = H_cache, D_cache
        an.run(hs, ds, sts, sus)
        return hs, ds

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = _lib.launch_count()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xff)                 # evict L2 (126 MB) outside the timed events
            starts[i].record(stream)
            step(kev[i])
            ends[i].record(stream)
            seg_total.add_(tr.stats[:, 1].sum())     # after the end event: not timed
            tail_total.add_(tr.stats[:, 9].sum())    # EF_ST_TAIL
            work_total.add_(tr.stats[:, [7, 8, 3]].sum(0))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n_launch = _lib.launch_count() - n_launch0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = sum(step_ms)
    k_ms = sum(a.elapsed_time(b) for a, b in kev)
    segs_per_step = int(seg_total.item()) / args.steps   # this rank's mean segments per frame
    tail_segs = int(tail_total.item()) / args.steps
    nodes_step, tris_step, arr_step = (int(x) / args.steps for x in work_total.cpu())
    arrivals = arr_step

    # ---- e2e through the public API: pinned host in/out, copies timed
    src_host = torch.from_numpy(np.ascontiguousarray(w.sources, np.float64)).pin_memory()
    # the step's result: the LowRateIR (histogram + direct block) of each of
    # this rank's sources -- what trace_frame returns --
    # plus the per-(source, band) reverb parameters and per-source predelay /
    # mean free path
    H_host = torch.empty((S_own,) + tuple(tr.H.shape[1:]), dtype=torch.float32).pin_memory()
    D_host = torch.empty((S_own,) + tuple(tr.Dir.shape[1:]), dtype=torch.float32).pin_memory()
    P_host = torch.empty(tuple(an.params.shape), dtype=torch.float64).pin_memory()
    Q_host = torch.empty(tuple(an.src_params.shape), dtype=torch.float64).pin_memory()
    e_starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e_ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    def e2e_step():
        tr.src_pos.copy_(src_host, non_blocking=True)
        hs, ds = step()
        H_host.copy_(hs, non_blocking=True)
        D_host.copy_(ds, non_blocking=True)
        P_host.copy_(an.params, non_blocking=True)
        Q_host.copy_(an.src_params, non_blocking=True)

    pipelined = world == 1 and not dynamic and big_inputs
    if pipelined:
        # Frame i's read-back (a copy stream) overlaps frame i+1's trace: two
        # tracer / analyzer / pinned-buffer slots, the timed span from the
        # first upload to the last read-back.  No L2 flush: the frame's
        # inputs exceed the L2 (scene + histograms, `big_inputs`).
        tr2 = FrameTracer(sc, S, cfg)
        tr2.set_sources(w.sources)
        an2 = Analyzer(S_own, w.n_bins, sc.n_bands, w.order, w.bin_s)
        hosts = [(H_host, D_host, P_host, Q_host),
                 tuple(torch.empty_like(x).pin_memory() for x in (H_host, D_host, P_host, Q_host))]
        slots = [(tr, an), (tr2, an2)]
        copy_st = torch.cuda.Stream()
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [torch.cuda.Event(), torch.cuda.Event()]

        def run_pipelined(n, t0=None, t1=None):
            if t0 is not None:
                t0.record(stream)
            for i in range(n):
                k = i & 1
                trk, ank = slots[k]
                if i >= 2:
                    stream.wait_event(freed[k])           # slot k's last read-back done
                trk.src_pos.copy_(src_host, non_blocking=True)
                trk.trace(w.listener, frame=i % max(w.n_frames, 1))
                ank.run(trk.H, trk.Dir, trk.stats, trk.sum_t)
                ready[k].record(stream)
                copy_st.wait_event(ready[k])
                with torch.cuda.stream(copy_st):
                    for dst, src in zip(hosts[k], (trk.H, trk.Dir, ank.params, ank.src_params)):
                        dst.copy_(src, non_blocking=True)
                    freed[k].record(copy_st)
            stream.wait_stream(copy_st)
            if t1 is not None:
                t1.record(stream)

        run_pipelined(args.warmup)
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        host_t0 = time.perf_counter()
        run_pipelined(args.steps, t0, t1)
        host_enqueue_ms = (time.perf_counter() - host_t0) * 1e3 / args.steps
        torch.cuda.synchronize()
        e_ms = t0.elapsed_time(t1)
        del tr2, an2
    else:
        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize()
        host_t0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            e_starts[i].record(stream)
            e2e_step()
            e_ends[i].record(stream)
        host_enqueue_ms = (time.perf_counter() - host_t0) * 1e3 / args.steps
        torch.cuda.synchronize()
        e_ms = sum(s.elapsed_time(e) for s, e in zip(e_starts, e_ends))
    h2d = src_host.numel() * 8
    d2h = H_host.numel() * 4 + D_host.numel() * 4 + P_host.numel() * 8 + Q_host.numel() * 8

    # ---- max over ranks, totals over ranks
    t = torch.tensor([ms, k_ms, e_ms], dtype=torch.float64, device=dev)
    segs = torch.tensor([float(seg_total.item())], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(segs, op=dist.ReduceOp.SUM)
    ms, k_ms, e_ms = (float(x) for x in t.cpu())
    total_segs = float(segs.item())
    value = total_segs / (ms * 1e-3)
    e2e_value = total_segs / (e_ms * 1e-3)

    # ---- roofline of the dominant kernel (trace): algorithmic bytes / launch
    peak, peak_kind = measured_peaks()
    bseg = b_seg(args.config, sc.n_bands, nk)
    avg_k_s = (k_ms * 1e-3) / args.steps
    achieved = bseg * segs_per_step / avg_k_s / 1e9
    # DRAM bytes of the trace call from the committed ncu captures: the trace
    # kernel plus, where the scene has one, the frame's tail kernel
    traffic = None
    ncu_util = None
    for suffix in ("", "tail"):
        tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}{suffix}.json")
        if os.path.exists(tf):
            with open(tf) as f:
                tj = json.load(f)
            traffic = (traffic or 0.0) + tj.get("dram_bytes_per_launch")
            if not suffix:
                ncu_util = tj.get("utilisation")
    if world > 1:
        if fused:
            peers.close()
        else:
            nccl_ex.close()
        dist.barrier()
        dist.destroy_process_group()   # every rank tears NCCL down before exit
    if rank != 0:
        return
    # device-work roofline: the bytes the device kernels themselves touch per
    # segment (their own counters: 64-byte quantized 4-wide nodes visited,
    # 80 bytes of each triangle record tested, one 48-byte shading record +
    # two f32 factor rows per segment, a histogram read-modify-write per
    # arrival), against the measured L2 bandwidth (tools/micro/cache_bw.cu,
    # profiles/micro_peaks.json): the working set is L1/L2-resident.  What
    # binds the kernel is in "ncu": issue-slot, ALU-pipe and L1/TEX
    # utilisation of the committed capture (profiles/traffic_<config>.json)
    dev_bytes = (64.0 * nodes_step + 80.0 * tris_step + (48 + 8 * sc.n_bands) * segs_per_step
                 + arr_step * 8 * sc.n_bands * nk)
    micro = {}
    mp = os.path.join(ROOT, "profiles", "micro_peaks.json")
    if os.path.exists(mp):
        with open(mp) as f:
            micro = json.load(f)
    dev_achieved = dev_bytes / avg_k_s / 1e9
    roof_dev = {"bound": "l2", "achieved": dev_achieved, "unit": "GB/s",
                "peak": micro.get("l2_read_gbs"), "l1_peak": micro.get("l1_read_gbs"),
                "frac": dev_achieved / micro["l2_read_gbs"] if micro.get("l2_read_gbs") else None,
                "bytes_per_segment": dev_bytes / max(segs_per_step, 1.0),
                "nodes_per_segment": nodes_step / max(segs_per_step, 1.0),
                "triangles_per_segment": tris_step / max(segs_per_step, 1.0),
                "peak_source": "profiles/micro_peaks.json (tools/micro/cache_bw.cu)" if micro else None,
                "ncu": ncu_util}
    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, w, world, "fused" if fused else "nccl"),
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms / args.steps,
                    "host_enqueue_ms_per_step": host_enqueue_ms,
                    "pipelining": ("frame i's IR read-back on a copy stream overlaps frame i+1's trace "
                                   "(two buffer slots); span from the first upload to the last read-back; "
                                   "no L2 flush (inputs > L2)") if pipelined else
                                  "serial per step (upload, trace, analysis, read-back), L2 flushed between steps"},
            "gpu_launches": int(n_launch),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": "trace_kernel" + (" + tail_kernel" if 512 < sc.n_triangles <= 4096 else ""),
                         "kernel_ms_per_launch": avg_k_s * 1e3,
                         "algorithmic_bytes_per_segment": bseg,
                         "segments_per_launch": round(segs_per_step)},
            "step_ms_quantiles": {q: float(np.percentile(step_ms, p)) for q, p in
                                  (("p10", 10), ("p50", 50), ("p90", 90), ("max", 100))},
            "roofline_device": roof_dev,
            "segments_per_step": total_segs / args.steps, "arrivals_per_step": arrivals,
            "tail_segments_per_step": tail_segs,
            "clocks": clocks.summary()}
    if exchange_note:
        line["exchange_note"] = exchange_note
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        rays = max(1, int(w.n_rays * args.cpu_fraction))
        rate, segs_c, dt, frames = cpu_oracle_rate(w, rays, cores, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": unit, "cores": cores, "kind": "port",
                                "sample": f"{frames} frames x rays [0,{rays}) of each of the "
                                          f"{len(w.sources)} sources ({segs_c} segments, {dt:.1f} s, "
                                          f"{cores} threads)"}
    print(json.dumps(line), flush=True)


def run_inflight(args, w, metric, unit):
    """Frames in flight (one GPU, static configs): F FrameTracer/Analyzer
    sets on F streams, frame i on set i % F, so frame i+1's trace kernel
    takes the SMs that frame i's tail releases (C2: one 100-bounce path keeps
    ~1/3 of a lone frame busy on one SM).  Throughput = all
    segments / the span of the K timed frames (CUDA events); per-frame
    latency = each frame's own start -> end events.  The L2 is not flushed
    between frames here (they overlap); the C2 scene (0.3 MB) is L1/L2
    resident either way.  e2e repeats with per-frame host copies (source
    positions in; LowRateIR + parameters out, pinned, per slot)."""
    import torch

    from paper_1803_00430_b200 import _lib
    from paper_1803_00430_b200.analysis import Analyzer
    from paper_1803_00430_b200.propagation import FrameTracer, TraceConfig
    from paper_1803_00430_b200.scene import scene_from_workload

    world, rank, local = dist_env()
    if world != 1:
        raise SystemExit("--inflight is a single-GPU mode")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    F = args.inflight
    sc = scene_from_workload(w)
    S = len(w.sources)
    cfg = TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                      bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius, seed=w.seed)
    slots = []
    for _ in range(F):
        tr = FrameTracer(sc, S, cfg)
        tr.set_sources(w.sources)
        an = Analyzer(S, w.n_bins, sc.n_bands, w.order, w.bin_s)
        host = {"src": torch.from_numpy(np.ascontiguousarray(w.sources, np.float64)).pin_memory(),
                "H": torch.empty(tuple(tr.H.shape), dtype=torch.float32).pin_memory(),
                "D": torch.empty(tuple(tr.Dir.shape), dtype=torch.float32).pin_memory(),
                "P": torch.empty(tuple(an.params.shape), dtype=torch.float64).pin_memory(),
                "Q": torch.empty(tuple(an.src_params.shape), dtype=torch.float64).pin_memory()}
        slots.append((torch.cuda.Stream(), tr, an, host, torch.zeros((), dtype=torch.int64, device=dev)))
    nf = max(w.n_frames, 1)

    def frame(i, ev=None, e2e=False):
        st, tr, an, host, segs = slots[i % F]
        with torch.cuda.stream(st):
            if ev is not None:
                ev[0].record(st)
            if e2e:
                tr.src_pos.copy_(host["src"], non_blocking=True)
            tr.trace(w.listener, frame=i % nf, stream=st)
            an.run(tr.H, tr.Dir, tr.stats, tr.sum_t, stream=st)
            if e2e:
                host["H"].copy_(tr.H, non_blocking=True)
                host["D"].copy_(tr.Dir, non_blocking=True)
                host["P"].copy_(an.params, non_blocking=True)
                host["Q"].copy_(an.src_params, non_blocking=True)
            if ev is not None:
                ev[1].record(st)
            segs.add_(tr.stats[:, 1].sum())

    def timed(e2e):
        for i in range(args.warmup):
            frame(i, e2e=e2e)
        torch.cuda.synchronize()
        for sl in slots:
            sl[4].zero_()
        n0 = _lib.launch_count()
        main = torch.cuda.current_stream()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        t0.record(main)
        for sl in slots:
            sl[0].wait_event(t0)
        for i in range(args.steps):
            frame(args.warmup + i, evs[i], e2e)
        for sl in slots:
            main.wait_stream(sl[0])
        t1.record(main)
        torch.cuda.synchronize()
        span = t0.elapsed_time(t1)
        lat = [a.elapsed_time(b) for a, b in evs]
        segs = sum(int(sl[4].item()) for sl in slots)
        return span, lat, segs, _lib.launch_count() - n0

    with ClockSampler(local) as clocks:
        span, lat, segs, n_launch = timed(False)
    e_span, e_lat, e_segs, _ = timed(True)
    st0, tr0, an0, host0, _ = slots[0]
    h2d = host0["src"].numel() * 8
    d2h = host0["H"].numel() * 4 + host0["D"].numel() * 4 + host0["P"].numel() * 8 + host0["Q"].numel() * 8
    value = segs / (span * 1e-3)
    peak, peak_kind = measured_peaks()
    bseg = b_seg(args.config, sc.n_bands, cfg.n_coeffs)
    achieved = bseg * segs / (span * 1e-3) / 1e9
    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": span / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_block(args, w, 1), frames_in_flight=F,
                           l2="not flushed: frames overlap (scene L1/L2-resident)"),
            "e2e": {"value": e_segs / (e_span * 1e-3), "unit": unit, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e_span / args.steps},
            "gpu_launches": int(n_launch),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_kind,
                         "kernel": "trace_kernel + tail_kernel (frames overlapped; span time)",
                         "algorithmic_bytes_per_segment": bseg},
            "frame_latency_ms": {q: float(np.percentile(lat, p)) for q, p in
                                 (("p10", 10), ("p50", 50), ("p90", 90), ("max", 100))},
            "segments_per_step": segs / args.steps, "clocks": clocks.summary()}
    print(json.dumps(line), flush=True)


def run_c4(args):
    """C4: sources rendered per 512-sample block within the 10.667 ms
    deadline (BASELINE configs[3]).  Sweeps S geometrically, then bisects
    between the last passing and first failing count; one step = one block
    for all S sources (crossover, taps, FDN, SH bus, binaural)."""
    import torch

    from paper_1803_00430_b200 import _lib, render, workloads
    world, rank, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    deadline_ms = 512 / 48000 * 1e3
    base = workloads.c4_params(n_sources=64)
    free, total = torch.cuda.mem_get_info()
    per_src = 4 * 8192 * 4 + 4 * 16 * 4096 * 4 + 4 * 4 * 16 * 16 + 2048 + 512   # C4 delays fit an 8192 ring
    s_cap = int(0.85 * free / per_src)

    def params(S):
        reps = (S + 63) // 64
        out = {}
        for k, v in base.items():
            if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == 64:
                out[k] = np.concatenate([v] * reps)[:S]
            else:
                out[k] = v
        return out

    # the configured input: seeded pink noise (workloads.pink_noise), 64
    # distinct source signals tiled over S sources, one 512-sample block
    pink = torch.from_numpy(workloads.pink_noise(64, 3 * 512))

    def pink_block(S, k=0):
        reps = (S + 63) // 64
        return pink[:, k * 512:(k + 1) * 512].repeat(reps, 1)[:S].contiguous()

    def measure(S, steps):
        r = render.SHRenderer(params(S))
        x = pink_block(S).to(dev)
        for _ in range(args.warmup):
            r.process(x, want_bus=False)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        n0 = _lib.launch_count()
        for a, b in ev:
            a.record()
            r.process(x, want_bus=False)
            b.record()
        torch.cuda.synchronize()
        ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        launches = _lib.launch_count() - n0
        # e2e: each block's audio uploaded from pinned host memory and the
        # binaural block read back, as a real-time host runs it: block k+1's
        # upload (copy stream, double-buffered input) overlaps block k's
        # render, so the period is max(upload, render + read-back) and the
        # output is one block later.  Every upload and read-back is inside
        # the timed span (first upload to last read-back).
        xh = [pink_block(S, k).pin_memory() for k in (1, 2)]
        xd = [x, torch.empty_like(x)]
        oh = torch.empty((2, 512), dtype=torch.float32).pin_memory()
        main = torch.cuda.current_stream()
        cs = torch.cuda.Stream()
        ready = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(main)
        cs.wait_event(t0)
        with torch.cuda.stream(cs):
            xd[0].copy_(xh[0], non_blocking=True)
            ready[0].record(cs)
        for k in range(steps):
            cur, nxt = k & 1, (k + 1) & 1
            if k + 1 < steps:
                if k >= 1:
                    cs.wait_event(consumed[nxt])     # block k-1 no longer reads xd[nxt]
                with torch.cuda.stream(cs):
                    xd[nxt].copy_(xh[nxt], non_blocking=True)
                    ready[nxt].record(cs)
            main.wait_event(ready[cur])
            r.process(xd[cur], want_bus=False)
            oh.copy_(r.out, non_blocking=True)
            consumed[cur].record(main)
        t1.record(main)
        torch.cuda.synchronize()
        e2e_ms = t0.elapsed_time(t1) / steps
        del r, x, xd
        torch.cuda.empty_cache()
        return ms, e2e_ms, launches

    sweep = []
    S = 64
    last_ok = None
    first_bad = None
    with ClockSampler(local) as clocks:
        while S <= s_cap:
            ms, e2e_ms, launches = measure(S, args.steps)
            sweep.append({"sources": S, "ms_per_block": round(ms, 4), "e2e_ms_per_block": round(e2e_ms, 4)})
            if ms <= deadline_ms:
                last_ok = (S, ms, e2e_ms, launches)
                S *= 2
            else:
                first_bad = S
                break
        if first_bad is None and last_ok and last_ok[0] < s_cap:
            first_bad = s_cap + 1
        lo = last_ok[0] if last_ok else 0
        hi = first_bad if first_bad else lo
        for _ in range(4):
            if hi - lo <= max(64, lo // 32):
                break
            mid = (lo + hi) // 2
            if mid > s_cap:
                break
            ms, e2e_ms, launches = measure(mid, args.steps)
            sweep.append({"sources": mid, "ms_per_block": round(ms, 4), "e2e_ms_per_block": round(e2e_ms, 4)})
            if ms <= deadline_ms:
                lo, last_ok = mid, (mid, ms, e2e_ms, launches)
            else:
                hi = mid
    S_max, ms, e2e_ms, launches = last_ok
    # e2e: largest S whose host-in/host-out block also meets the deadline
    e2e_ok = [p["sources"] for p in sweep if p["e2e_ms_per_block"] <= deadline_ms]
    bytes_per_src = (8192 + 16384 + 2 * 16 * 4 * 512 * 4 + 4096 + 2048)   # DESIGN.md 5 (C4)
    achieved = bytes_per_src * S_max / (ms * 1e-3) / 1e9
    peak, kind = measured_peaks()
    line = {"metric": "sources rendered per audio block within the 10.667 ms deadline",
            "value": S_max, "unit": "sources/block", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "c4_auralization (BASELINE.json configs[3])", "block": 512,
                       "fs": 48000, "sh_order": 3, "fdn_lines_per_band": 16, "bands": 4,
                       "hrtf": "16x2 x 256 taps, overlap-save FFT 1024",
                       "memory_cap_sources": s_cap, "l2": "state > L2 (HBM-resident)"},
            "e2e": {"value": max(e2e_ok) if e2e_ok else 0, "unit": "sources/block",
                    "h2d_bytes_per_step": (max(e2e_ok) if e2e_ok else 0) * 512 * 4,
                    "d2h_bytes_per_step": 2 * 512 * 4,
                    "ms_per_step": min((p["e2e_ms_per_block"] for p in sweep
                                        if e2e_ok and p["sources"] == max(e2e_ok)), default=None),
                    "pipelining": "block k+1 uploaded on a copy stream during block k's render "
                                  "(one block of extra latency)"},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": kind,
                         "kernel": "xover+render+reduce+bus", "algorithmic_bytes_per_source": bytes_per_src},
            "sweep": sweep, "clocks": clocks.summary()}
    if not args.no_cpu_baseline:
        from oracle import audio as OA4
        S_cpu = 8
        p8 = workloads.c4_params(n_sources=S_cpu)
        xs = workloads.pink_noise(S_cpu, 512 * 6)
        ora = OA4.AudioOracle(p8, p8["hrtf"])
        ora.process(xs[:, :512])
        t0 = time.perf_counter()
        for k in range(1, 6):
            ora.process(xs[:, k * 512:(k + 1) * 512])
        per_block = (time.perf_counter() - t0) / 5
        line["cpu_baseline"] = {"value": S_cpu * deadline_ms * 1e-3 / per_block, "unit": "sources/block",
                                "cores": 1, "kind": "port",
                                "sample": f"oracle/audio.py (f64 numpy) on {S_cpu} sources x 5 blocks, "
                                          f"{per_block * 1e3:.1f} ms per block"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default 10 (C5), 200 (others)")
    ap.add_argument("--warmup", type=int, default=None, help="default 3 (C5), 10 (others)")
    ap.add_argument("--config", default="c5", choices=sorted(WORK) + ["c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-fraction", type=float, default=None,
                    help="fraction of each source's rays in the CPU sample (default per config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N > 1: histogram reduce-scatter inside the trace kernel over peer "
                         "memory (fused) or a separate NCCL reduce-scatter")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: several ranks on one GPU for plumbing checks (fused only)")
    ap.add_argument("--inflight", type=int, default=1,
                    help="frames in flight on separate streams (single GPU, static configs)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="minimum wall time of the CPU baseline sample")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 10 if args.config == "c5" else 200
    if args.warmup is None:
        args.warmup = 3 if args.config == "c5" else 10
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    from paper_1803_00430_b200 import workloads
    if args.config == "c4":
        args.steps = min(args.steps, 20)
        return run_c4(args)
    w = workloads.WORKLOADS[args.config]()
    if args.cpu_fraction is None:
        args.cpu_fraction = {"c1": 1.0, "c2": 1.0, "c3": 1.0 / 32, "c5": 1.0 / 1024}[args.config]
    metric = "ray-bounce segments/sec into SH energy IRs"
    unit = "segments/s"
    if args.impl == "reference":
        run_reference(args, w, metric, unit)
    elif args.inflight > 1:
        if w.n_frames > 1 and w.source_velocity is not None:
            raise SystemExit("--inflight needs a static config (C3's frames are sequential)")
        run_inflight(args, w, metric, unit)
    else:
        run_gpu(args, w, metric, unit)


if __name__ == "__main__":
    main()

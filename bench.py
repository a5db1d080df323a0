#!/usr/bin/env python
"""Benchmark of the read-mapping hot path: reads/s mapped per B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

One step = one read buffer (config C2 by default: 1M simulated 100 bp reads at
3% edits against a 100 Mbp random reference, q=16, all-hits mode, band 32, 80%
identity) through index build -> filtration -> candidate sort/unique ->
banded Myers validation -> dedup/strata.

* value    : reads in HBM (2-bit words) when the step starts; step = read prep
             (device-to-device copy + bit planes) + qgm_map; CUDA events on the
             library's stream, per step, L2 flushed between steps (a 512 MiB
             write, outside the step's events). Sum of the K step times, max
             over ranks.
* e2e      : the public C ABI from pinned host buffers, K steps = K read
             batches through qgm_map_host_batches (the streamed run_map
             pipeline: batch i+1's H2D and batch i-1's hit D2H overlap batch
             i's mapping on a second stream); every step copies its reads in
             and its hits out. CUDA events around the K-batch call. The step's
             working set (3.2 GB reference index, 0.7 GB items) exceeds L2,
             so no flush is needed between its steps. `e2e_unpipelined` is the
             one-call-per-batch qgm_map_host for comparison.
* roofline : the dominant kernel of the step (largest CUDA-event time among
             the hot kernels), algorithmic bytes per launch (DESIGN.md section
             4) / its measured launch time, against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline (rank 0, N=1): the reference's build_qgroup_index + the oracle
             restatement of stages 2-5 (oracle/_ref/libqgm_ref.so) on the host
             cores, on one full C2 batch.
Multi-GPU (torchrun): reads are sharded -- every rank maps its own 1M-read
batch against its own copy of the reference (weak scaling, no data-path
collective); NCCL only carries the barrier and the max-over-ranks timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reads/sec mapped (100 bp, best & all mode) at 1/2/4/8 B200 vs host-CPU ref"

CONFIGS = {
    # name: (ref_bp, n_chrom, reads, read_len, err, q, mode, band, pct, repetitive)
    "C1": (1_000_000, 1, 10_000, 100, 0.03, 12, 0, 32, 80, False),
    "C2": (100_000_000, 1, 1_000_000, 100, 0.03, 16, 1, 32, 80, False),
    "C2q12": (100_000_000, 1, 1_000_000, 100, 0.03, 12, 1, 32, 80, False),
    "C3": (3_100_000_000, 24, 1_250_000, 100, 0.03, 16, 0, 32, 80, False),
    "C4": (100_000_000, 1, 1_000_000, 250, 0.08, 16, 1, 32, 80, False),
    "C5": (100_000_000, 1, 1_000_000, 100, 0.03, 16, 1, 32, 80, True),
    "C5m": (100_000_000, 1, 1_000_000, 100, 0.03, 16, 1, 32, 80, True),
}
MASK_THRESHOLD = {"C5m": 1000}  # device repeat mask applied before the timed region
DESCR = {
    "C1": "C1: 1 Mbp random reference + 10k simulated 100 bp reads (3% edits), q=12, best-stratum",
    "C2": "C2: 100 Mbp random reference + 1M simulated 100 bp reads (3% edits), q=16, all-hits",
    "C2q12": "C2 at q=12 (stress): 100 Mbp + 1M 100 bp reads, all-hits",
    "C3": "C3 shard: 3.1 Gbp (24 chromosomes) + 1.25M 100 bp reads per GPU, q=16, best-stratum",
    "C4": "C4: 100 Mbp + 1M 250 bp reads at 8% edits, q=16, all-hits",
    "C5": "C5: 100 Mbp repetitive reference + 1M 100 bp reads, q=16, all-hits",
    "C5m": "C5 with the repeat mask at threshold 1000 (SPEC.md:302): 100 Mbp repetitive reference + 1M 100 bp reads, "
           "q=16, all-hits",
}


def chrom_begin(total, n):
    if n == 1:
        return np.array([0, total], np.uint64)
    # human-like decreasing chromosome lengths
    w = np.linspace(2.0, 0.5, n)
    lens = np.floor(w / w.sum() * total).astype(np.uint64)
    lens[-1] += np.uint64(total - int(lens.sum()))
    return np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every 200 ms in a
    background thread during the timed region (in-process NVML: no nvidia-smi
    subprocess contending for the driver while kernels are timed)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device, period=0.2):
        self.device, self.period = device, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = None

    def _run(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.reasons |= {k for k, v in self.REASONS.items() if mask & v}
            self._stop.wait(self.period)

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            self._nvml_index = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._stop = None
        return self

    def __exit__(self, *a):
        if self._stop:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


def make_inputs(qgm, cfg, rank):
    ref_bp, n_chrom, n_reads, rlen, err, q, mode, band, pct, rep = cfg
    ref = qgm.repetitive_reference(7, ref_bp) if rep else qgm.random_reference(7, ref_bp)
    cb = chrom_begin(ref_bp, n_chrom)
    codes, lengths, *_ = qgm.simulate_reads(1000 + rank, ref, cb, n_reads, rlen, err)
    return ref, cb, codes, lengths


def algorithmic_bytes(kernel, cfg, st, ref_bp, n_reads):
    """Algorithmic HBM bytes of one launch of `kernel` (DESIGN.md section 4 /
    SURVEY.md section 8(d))."""
    q, rlen = cfg[5], cfg[3]
    groups = (4 ** q) // 32
    V, D = st["index_occurrences"], st["index_distinct"]
    if kernel == "k_filter":
        n_look = 2 * (ref_bp - q + 1)
        return ref_bp / 4 + 4 * n_look + 12 * st["lookups_hit"] + 4 * st["occurrences"] + 8 * st["raw_candidates"]
    if kernel == "k_join":
        # canonical-code join (join.cu): read join items (8 B) + the occupancy
        # words (4 B) and u16 group starts (2 B) of the one canonical index,
        # each once + the two S' entries per lookup hit + one O word per
        # occurrence visited + 8 B per candidate key written
        return 8 * V + 6 * groups + 8 * st["lookups_hit"] + 4 * st["occurrences"] + 8 * st["raw_candidates"]
    if kernel == "k_part_hist":
        return n_reads * rlen / 4 + 4 * n_reads
    if kernel in ("k_part_scatter", "k_refine_scatter"):
        return (n_reads * rlen / 4 + 4 * n_reads if kernel == "k_part_scatter" else 8 * V) + 8 * V
    if kernel == "k_refine_hist":
        return 8 * V
    if kernel == "k_hash_insert":
        return 8 * st["raw_candidates"] + 8 * st["unique_candidates"]
    if kernel == "k_bucket_rank":
        return n_reads * rlen / 4 + 4 * V
    if kernel == "k_bucket_scatter":
        return n_reads * rlen / 4 + 4 * V + 8 * V
    if kernel == "k_bucket_occupy":
        return 8 * V + 4 * groups
    if kernel == "k_bucket_emit":
        return 16 * V + 4 * groups + 4 * (groups + 1) + 4 * (D + 1) + 4 * V
    if kernel == "radix_sort_keys":
        return 8 * st["raw_candidates"] + 8 * st["unique_candidates"]
    if kernel == "k_validate":
        u = st["unique_candidates"]
        return u * (8 + rlen / 4 + (rlen + cfg[7] - 1) / 4 + 12)
    return None


def bind_to_gpu_numa(local):
    """Run this rank on the host cores NVML reports as local to its GPU, so the
    pinned read/hit buffers live on the GPU's NUMA node (PCIe copies do not
    cross sockets). Returns the core count, or None when NVML is unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = int(vis.split(",")[local]) if vis and vis.split(",")[0].isdigit() else local
        h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        n_words = (os.cpu_count() + 63) // 64
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, n_words)
        cpus = {64 * w + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        return None
    return None


def run_gpu(args):
    import torch
    import paper_1403_1706_b200 as qgm

    from paper_1403_1706_b200 import sharding

    rank, world, local = sharding.world()
    numa_cores = bind_to_gpu_numa(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    cfg = CONFIGS[args.config]
    ref_bp, n_chrom, n_reads, rlen, err, q, mode, band, pct, rep = cfg
    ref, cb, codes, lengths = make_inputs(qgm, cfg, rank)
    stream = torch.cuda.Stream(local)
    ctx = qgm.Context(local, stream=stream.cuda_stream)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    t0 = time.perf_counter()
    if args.config in MASK_THRESHOLD:
        R.mask_repeats(q, MASK_THRESHOLD[args.config])
    R.prepare(q)  # reference preprocessing (once per reference and q), outside every timed region
    ref_prepare_s = time.perf_counter() - t0
    words = qgm.pack_read_codes(codes, rlen)
    params = qgm.make_params(q=q, mode=mode, band_width=band, pct_identity=pct)
    lib = ctx.lib
    import ctypes as C

    # device-resident inputs for `value`
    d_words = torch.from_numpy(words.view(np.int64)).to(f"cuda:{local}")
    d_len = torch.from_numpy(lengths.view(np.int32)).to(f"cuda:{local}")
    # pinned host inputs / outputs for `e2e`, allocated before anything else
    # large (placement of pinned pages allocated late in the process varied
    # the streamed time by up to 20% between processes on one box)
    # the streamed API takes the reads as one dense 2-bit stream (2 bits per
    # base, no per-read padding) and, all reads being `rlen` long, no length
    # array: 25 MB per 1M x 100 bp batch
    uniform = bool(np.all(lengths == rlen))
    h_dense = torch.from_numpy(qgm.pack_codes(codes).view(np.int64)).pin_memory()
    h_words = torch.from_numpy(words.view(np.int64)).pin_memory()
    h_len = torch.from_numpy(lengths.view(np.int32)).pin_memory()
    cap = n_reads * 4  # resized from the measured hit count before the e2e pass
    h_hits = torch.empty(cap * 16, dtype=torch.uint8).pin_memory()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def step_device():
        rd = C.c_void_p()
        ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(d_words.data_ptr()), C.c_void_p(d_len.data_ptr()),
                                             n_reads, rlen, C.byref(rd)))
        h = C.c_void_p()
        ctx._check(lib.qgm_map(ctx.h, rd, R.h, C.byref(params), C.byref(h)))
        st = qgm.MapStats()
        lib.qgm_hits_stats(h, C.byref(st))
        lib.qgm_hits_destroy(h)
        lib.qgm_reads_destroy(rd)
        return {f: getattr(st, f) for f, _ in qgm.MapStats._fields_}

    def step_e2e():
        n = C.c_uint64()
        st = qgm.MapStats()
        ctx._check(lib.qgm_map_host(ctx.h, C.c_void_p(h_words.data_ptr()), C.c_void_p(h_len.data_ptr()), n_reads,
                                    rlen, R.h, C.byref(params), C.c_void_p(h_hits.data_ptr()), cap, C.byref(n),
                                    C.byref(st)))
        return n.value

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, K, with_profile=False):
        times = []
        out = None
        launches = 0
        for _ in range(K):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.launches(reset=True)
            out = fn()
            launches += ctx.launches()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return times, out, launches

    for _ in range(args.warmup):
        step_device()
    barrier()
    with ClockSampler(local, period=args.clock_period) as clk:
        times, st, launches = timed(step_device, args.steps)
        barrier()
    clocks = clk.summary()
    dev_ms = sum(times)
    # pinned hit output sized from the device pass's hit count
    if st["hits"] > cap:
        cap = int(st["hits"] * 1.05) + 1024
        h_hits = torch.empty(cap * 16, dtype=torch.uint8).pin_memory()

    def run_batches(K):
        arr = (qgm.Batch * K)()
        for i in range(K):
            arr[i] = qgm.Batch(h_dense.data_ptr(), None if uniform else h_len.data_ptr(), n_reads, rlen,
                               h_hits.data_ptr(), cap, 0, qgm.MapStats(), qgm.READS_DENSE, 0)
        ctx._check(lib.qgm_map_host_batches(ctx.h, arr, K, R.h, C.byref(params)))
        return arr[K - 1].n_out

    run_batches(max(args.steps, args.warmup, 3))  # warm-up with the timed batch count
    barrier()
    # three timed runs of the K pipelined batches; the median is reported
    # (host-side jitter moves single runs by up to ~10%)
    e2e_runs = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_hits = run_batches(args.steps)
        e1.record(stream)
        e1.synchronize()
        barrier()
        e2e_runs.append(e0.elapsed_time(e1))
    e2e_ms = sorted(e2e_runs)[1]
    e2e_times = [round(t / args.steps, 3) for t in e2e_runs]

    # one qgm_map_host call per batch, for comparison
    for _ in range(max(1, args.warmup // 2)):
        step_e2e()
    barrier()
    e2e1_times, n_hits, _ = timed(step_e2e, args.steps)
    barrier()
    e2e1_ms = sum(e2e1_times)

    # profile pass (per-kernel CUDA events; not part of `value`)
    ctx.profile(True)
    ctx.kernel_times(reset=True)
    ctx.stage_times(reset=True)
    prof_steps = max(1, min(3, args.steps))
    timed(step_device, prof_steps)
    ktimes = ctx.kernel_times(reset=True)
    stimes = ctx.stage_times(reset=True, host=True)
    ctx.profile(False)
    post = postprocess_pass(ctx, lib, C, qgm, R, d_words, d_len, n_reads, rlen, params, band)
    dev_ms, e2e_ms, e2e1_ms = sharding.max_over_ranks([dev_ms, e2e_ms, e2e1_ms], dist, device=f"cuda:{local}")
    total_reads = n_reads * args.steps * world
    value = sharding.weak_scaling_value(n_reads, args.steps, world, dev_ms)
    e2e_value = sharding.weak_scaling_value(n_reads, args.steps, world, e2e_ms)
    e2e1_value = sharding.weak_scaling_value(n_reads, args.steps, world, e2e1_ms)

    # roofline of the dominant kernel
    peak, peak_kind = load_peaks()
    per_launch = {k: v[0] / v[1] for k, v in ktimes.items()}
    dom = max(per_launch, key=per_launch.get) if per_launch else None
    roof = None
    if dom:
        ab = algorithmic_bytes(dom, cfg, st, ref_bp, n_reads)
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(dom)
        if ab is not None:
            ach = ab / (per_launch[dom] / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": traffic, "peak_source": peak_kind,
                    "algorithmic_bytes": int(ab), "launch_ms": round(per_launch[dom], 4),
                    "share_of_step": round(ktimes[dom][0] / prof_steps / (sum(times) / len(times)), 4)}
    # every timed kernel against its own bound (HBM bytes, or for the
    # INT-ALU-bound validation the warp-instruction issue rate: 4 per SM per
    # clock, instruction count from the committed ncu profile)
    stage_roof = {}
    for kname, ms in per_launch.items():
        ab = algorithmic_bytes(kname, cfg, st, ref_bp, n_reads)
        if ab is not None and kname != "k_validate":
            ach = ab / (ms / 1e3) / 1e9
            stage_roof[kname] = {"bound": "hbm", "achieved_gbs": round(ach, 1), "frac": round(ach / peak, 4)}
    if "k_validate" in per_launch:
        ip = os.path.join(ROOT, "profiles", f"instructions_{args.config}.json")
        inst = json.load(open(ip)).get("k_validate") if os.path.exists(ip) else None
        if inst:
            clk = (clocks.get("sm_mhz") or 1965) * 1e6
            peak_issue = 148 * 4 * clk
            ach = inst / (per_launch["k_validate"] / 1e3)
            stage_roof["k_validate"] = {"bound": "issue (INT ALU)", "achieved_warp_inst_per_s": round(ach / 1e9, 1),
                                        "peak": round(peak_issue / 1e9, 1), "unit": "G warp-inst/s",
                                        "frac": round(ach / peak_issue, 4),
                                        }
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "reads/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": DESCR[args.config], "reads_per_gpu": n_reads, "read_len": rlen, "ref_bp": ref_bp,
                   "chromosomes": n_chrom, "q": q, "mode": ("best-stratum", "all")[mode], "band": band,
                   "pct_identity": pct, "parallelism": f"read-sharded x{world} (reference replicated)",
                   "l2": "flushed between steps (512 MiB device write outside the step events)"},
        "e2e": {"value": round(e2e_value, 1), "unit": "reads/s", "ms_per_step": round(e2e_ms / args.steps, 3),
                "h2d_bytes_per_step": int((n_reads * rlen + 31) // 32 * 8 + (0 if uniform else lengths.nbytes)),
                "d2h_bytes_per_step": int(n_hits * 16),
                "api": "qgm_map_host_batches (streamed; copies overlap mapping; dense 2-bit reads)",
                "runs": 3, "statistic": "median of 3 timed runs of K batches"},
        "e2e_unpipelined": {"value": round(e2e1_value, 1), "unit": "reads/s", "ms_per_step": round(e2e1_ms / args.steps, 3),
                            "api": "qgm_map_host, one call per batch",
                            "h2d_bytes_per_step": int(words.nbytes + lengths.nbytes)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "stage_roofline": stage_roof,
        "clocks": clocks,
        "step_ms": [round(t, 3) for t in times],
        "e2e_step_ms": e2e_times,  # per-batch time of each of the three timed runs
        "stages_ms_per_step": {k: round(v / prof_steps, 4) for k, v in stimes.items() if v},
        "kernels_ms_per_launch": {k: round(v, 4) for k, v in per_launch.items()},
        "counts": st,
        "reference_prepare_s": round(ref_prepare_s, 3),
        "host_binding": {"cores": numa_cores, "rule": "NVML CPU affinity of the rank's GPU"},
        "postprocess": post,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        os.sched_setaffinity(0, set(range(os.cpu_count())))  # the CPU baseline gets every host core
        line["cpu_baseline"] = cpu_baseline(args, cfg, ref, cb, codes, lengths, samples=1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    del R
    ctx.close()
    if dist:
        dist.destroy_process_group()


def postprocess_pass(ctx, lib, C, qgm, R, d_words, d_len, n_reads, rlen, params, band):
    """SPEC.md:446-483 tail on one batch's device-resident hits (not part of
    `value`): hit_rank (k_rank_keys + radix sort + k_ranks) and
    traceback_cigar (k_cigar), kernel times from CUDA events, second of two
    runs."""
    rd = C.c_void_p()
    ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(d_words.data_ptr()), C.c_void_p(d_len.data_ptr()),
                                         n_reads, rlen, C.byref(rd)))
    h = C.c_void_p()
    try:
        ctx._check(lib.qgm_map(ctx.h, rd, R.h, C.byref(params), C.byref(h)))
        n = C.c_uint64()
        lib.qgm_hits_count(h, C.byref(n))
        n = n.value
        if n == 0:
            return None
        max_ops = 48
        ops = np.empty(n * max_ops, np.uint32)
        info = np.empty(n, qgm.CIGAR_DTYPE)
        ranks = np.empty(n, np.uint32)
        ctx.profile(True)
        for it in range(2):
            ctx.kernel_times(reset=True)
            ctx._check(lib.qgm_hits_ranks(ctx.h, h, C.c_void_p(ranks.ctypes.data)))
            st = lib.qgm_hits_cigar(ctx.h, h, rd, R.h, band, max_ops, C.c_void_p(ops.ctypes.data),
                                    C.c_void_p(info.ctypes.data))
            if st != 0:  # a record needs more operations
                max_ops = int(info["n_ops"].max())
                ops = np.empty(n * max_ops, np.uint32)
                ctx._check(lib.qgm_hits_cigar(ctx.h, h, rd, R.h, band, max_ops, C.c_void_p(ops.ctypes.data),
                                              C.c_void_p(info.ctypes.data)))
            kt = ctx.kernel_times(reset=True)
        ctx.profile(False)
        cig_ms = kt.get("k_cigar", (0.0, 1))[0]
        return {"hits": n, "k_cigar_ms": round(cig_ms, 4), "cigar_hits_per_s": round(n / (cig_ms / 1e3), 1),
                "cigar_ops_max": int(info["n_ops"].max()), "cigar_edits_mean": round(float(info["edits"].mean()), 3),
                "rank_ms": round(sum(v[0] for k, v in kt.items() if k != "k_cigar"), 4)}
    finally:
        if h:
            lib.qgm_hits_destroy(h)
        lib.qgm_reads_destroy(rd)


def cpu_baseline(args, cfg, ref, cb, codes, lengths, samples=1):
    """The reference's build_qgroup_index + restated stages 2-5 on the host cores."""
    from oracle.pyoracle import RefShim, Oracle, REF_SO, repeat_mask
    ref_bp, n_chrom, n_reads, rlen, err, q, mode, band, pct, rep = cfg
    threads = os.cpu_count() or 1
    kind = "reference" if os.path.exists(REF_SO) else "port"
    impl = RefShim() if kind == "reference" else Oracle()
    mask = repeat_mask(ref, cb, q, MASK_THRESHOLD[args.config]) if args.config in MASK_THRESHOLD else None
    times = []
    st = None
    for _ in range(samples):
        t0 = time.perf_counter()
        hits, st = impl.map(ref, cb, codes, rlen, lengths, q=q, mode=mode, band=band, pct=pct, threads=threads,
                            mask=mask)
        times.append(time.perf_counter() - t0)
    best = min(times)
    return {"value": round(n_reads / best, 1), "unit": "reads/s", "cores": threads, "kind": kind,
            "sample": f"one full {args.config} batch ({n_reads} reads vs {ref_bp} bp); "
                      f"index = reference build_qgroup_index (qgroup_index.hpp:124-180), stages 2-5 = oracle "
                      f"restatement; best of {samples}, {best:.2f} s", "hits": int(hits.size), "counts": st}


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores, rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import paper_1403_1706_b200 as qgm
    cfg = CONFIGS[args.config]
    ref, cb, codes, lengths = make_inputs(qgm, cfg, 0)
    from oracle.pyoracle import RefShim, Oracle, REF_SO, repeat_mask
    ref_bp, n_chrom, n_reads, rlen, err, q, mode, band, pct, rep = cfg
    threads = os.cpu_count() or 1
    kind = "reference" if os.path.exists(REF_SO) else "port"
    impl = RefShim() if kind == "reference" else Oracle()
    mask = repeat_mask(ref, cb, q, MASK_THRESHOLD[args.config]) if args.config in MASK_THRESHOLD else None
    for _ in range(args.warmup):
        impl.map(ref, cb, codes, rlen, lengths, q=q, mode=mode, band=band, pct=pct, threads=threads, mask=mask)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        hits, st = impl.map(ref, cb, codes, rlen, lengths, q=q, mode=mode, band=band, pct=pct, threads=threads,
                            mask=mask)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n_reads * args.steps / total
    line = {"metric": METRIC, "value": round(value, 1), "unit": "reads/s", "n_gpus": int(os.environ.get("WORLD_SIZE", 1)),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": DESCR[args.config], "reads_per_step": n_reads, "ref_bp": ref_bp, "q": q,
                       "mode": ("best-stratum", "all")[mode]},
            "cpu_baseline": {"value": round(value, 1), "unit": "reads/s", "cores": threads, "kind": kind,
                             "sample": f"{args.steps} full {args.config} batches; index = reference "
                                       f"build_qgroup_index, stages 2-5 = oracle restatement (no reference code)"},
            "e2e": {"value": round(value, 1), "unit": "reads/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "counts": st, "hits": int(hits.size)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--clock-period", type=float, default=0.005, help="NVML clock sampling period (s)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

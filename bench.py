#!/usr/bin/env python
"""Benchmark of the read-mapping hot path: reads/s mapped on 1..N B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]
                    [--check off|sample|full] [--no-cpu]

One step = every read batch a rank maps in one pass of the hot path (index
build -> filtration -> candidate dedup -> banded Myers validation ->
dedup/strata). Configs (BASELINE.json): C1 1 Mbp / 10k reads / q=12 / best;
C2 (default) 100 Mbp / 1M reads / q=16 / all; C3 3.1 Gbp (24 chromosomes) /
10M reads / best, the job split over the ranks (strong scaling, 1.25M-read
batches); C4 250 bp at 8% (B=32, C4b64: B=64); C5 repetitive (C5m: repeat
mask 1000). Reads are blocks of simulated batches (block b: seed 1000+b), so a
job's reads do not depend on how many ranks map them.

* value   : reads in HBM (2-bit words) when the step starts; per batch read
            prep (device-to-device copy + bit planes) + qgm_map; CUDA events on
            the library's stream; L2 flushed between steps (a 512 MiB write
            outside the events); sum of the K step times, max over ranks.
* e2e     : the public C ABI from pinned host buffers: the K steps' batches
            through qgm_map_host_batches (H2D of batch i+1 and D2H of batch
            i-1's hits overlap batch i's mapping), then -- N > 1 -- the
            end-of-run gather of every rank's hits into one host buffer
            (sharding.HostGather). Median of 3 timed runs, max over ranks.
* roofline: the dominant kernel (largest per-launch CUDA-event time),
            algorithmic bytes per launch / launch time,
            against MEASURED_PEAKS.json; `traffic` = ncu DRAM bytes of that
            kernel from profiles/<round>/ncu_<config>.json when it was captured
            from a build of these exact sources and flags (`build_stamp`), else null.
* parity  : rank 0's first batch checked against the CPU path (reference
            build_qgroup_index + restated stages 2-5) in a SUBPROCESS (the GPU
            process never maps oracle/ code): digest of the sorted hit set of
            the first S reads (--check sample, S = the cpu_baseline sample) or
            of the whole batch (--check full).
* cpu_baseline (rank 0, N = 1): that subprocess's timing on all host cores,
            per stage, with the CPU model.
Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run (one process per GPU). NCCL when every rank has its own
GPU; with fewer GPUs than ranks (a 1-GPU box) the ranks share devices over
gloo ("oversubscribed": true -- a functional run, not a scaling number).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reads/sec mapped (100 bp, best & all mode) at 1/2/4/8 B200 vs host-CPU ref"
MODES = ("best-stratum", "all")


def _cfg(ref_bp, n_chrom, reads, batch, rlen, err, q, mode, band=32, pct=80, rep=False, mask=None, strong=False,
         cpu_sample=None, descr=""):
    return dict(ref_bp=ref_bp, n_chrom=n_chrom, reads=reads, batch=batch, rlen=rlen, err=err, q=q, mode=mode,
                band=band, pct=pct, repetitive=rep, mask_threshold=mask, strong=strong,
                cpu_sample=cpu_sample or batch, descr=descr)


CONFIGS = {
    "C1": _cfg(1_000_000, 1, 10_000, 10_000, 100, 0.03, 12, 0,
               descr="C1: 1 Mbp random reference + 10k simulated 100 bp reads (3% edits), q=12, best-stratum"),
    "C2": _cfg(100_000_000, 1, 1_000_000, 1_000_000, 100, 0.03, 16, 1, cpu_sample=500_000,
               descr="C2: 100 Mbp random reference + 1M simulated 100 bp reads (3% edits), q=16, all-hits"),
    "C2best": _cfg(100_000_000, 1, 1_000_000, 1_000_000, 100, 0.03, 16, 0, cpu_sample=500_000,
                   descr="C2 in best-stratum mode: 100 Mbp random reference + 1M 100 bp reads (3% edits), q=16"),
    "C2q12": _cfg(100_000_000, 1, 1_000_000, 1_000_000, 100, 0.03, 12, 1, cpu_sample=20_000,
                  descr="C2 at q=12 (stress): 100 Mbp + 1M 100 bp reads, all-hits"),
    "C3": _cfg(3_100_000_000, 24, 10_000_000, 1_250_000, 100, 0.03, 16, 0, strong=True, cpu_sample=50_000,
               descr="C3: 3.1 Gbp (24 chromosomes) + 10M 100 bp reads (3% edits), q=16, best-stratum, "
                     "reads sharded over the GPUs (1.25M-read batches)"),
    "C3shard": _cfg(3_100_000_000, 24, 1_250_000, 1_250_000, 100, 0.03, 16, 0, cpu_sample=50_000,
                    descr="C3 per-GPU shard: 3.1 Gbp (24 chromosomes) + 1.25M 100 bp reads per GPU, q=16, "
                          "best-stratum"),
    "C4": _cfg(100_000_000, 1, 1_000_000, 1_000_000, 250, 0.08, 16, 1, cpu_sample=100_000,
               descr="C4: 100 Mbp + 1M 250 bp reads at 8% edits, q=16, all-hits, band 32"),
    "C4b64": _cfg(100_000_000, 1, 1_000_000, 1_000_000, 250, 0.08, 16, 1, band=64, cpu_sample=100_000,
                  descr="C4 with band 64: 100 Mbp + 1M 250 bp reads at 8% edits, q=16, all-hits"),
    "C5": _cfg(100_000_000, 1, 1_000_000, 1_000_000, 100, 0.03, 16, 1, rep=True, cpu_sample=10_000,
               descr="C5: 100 Mbp repetitive reference + 1M 100 bp reads, q=16, all-hits, no mask"),
    "C5m": _cfg(100_000_000, 1, 1_000_000, 1_000_000, 100, 0.03, 16, 1, rep=True, mask=1000, cpu_sample=100_000,
                descr="C5 with the repeat mask at threshold 1000 (SPEC.md:302): 100 Mbp repetitive reference + "
                      "1M 100 bp reads, q=16, all-hits"),
}


def config_dict(name, cfg, world):
    """The `config` object of BOTH arms' JSON lines (identical by construction)."""
    return {"workload": cfg["descr"], "name": name, "ref_bp": cfg["ref_bp"], "chromosomes": cfg["n_chrom"],
            "reads_per_step": cfg["reads"] if cfg["strong"] else cfg["reads"] * world,
            "batch_reads": cfg["batch"], "read_len": cfg["rlen"], "edit_rate": cfg["err"], "q": cfg["q"],
            "mode": MODES[cfg["mode"]], "band": cfg["band"], "pct_identity": cfg["pct"],
            "repeat_mask": cfg["mask_threshold"], "scaling": "strong" if cfg["strong"] else "weak",
            "parallelism": f"reads sharded over {world} rank(s), reference replicated",
            "edit_model": "substitution/insertion/deletion 0.8/0.1/0.1, 50% reverse strand",
            "l2": "flushed between steps (512 MiB device write outside the step events)"}


def chrom_begin(total, n):
    if n == 1:
        return np.array([0, total], np.uint64)
    w = np.linspace(2.0, 0.5, n)  # human-like decreasing chromosome lengths
    lens = np.floor(w / w.sum() * total).astype(np.uint64)
    lens[-1] += np.uint64(total - int(lens.sum()))
    return np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)


def make_reference(qgm, cfg):
    ref = qgm.repetitive_reference(7, cfg["ref_bp"]) if cfg["repetitive"] else qgm.random_reference(7, cfg["ref_bp"])
    return ref, chrom_begin(cfg["ref_bp"], cfg["n_chrom"])


def make_block(qgm, cfg, ref, cb, block, n=None):
    """Read block `block` (seed 1000 + block): (codes, lengths); first n reads if given."""
    codes, lengths, *_ = qgm.simulate_reads(1000 + block, ref, cb, cfg["batch"], cfg["rlen"], cfg["err"])
    if n is not None and n < cfg["batch"]:
        codes, lengths = codes[: n * cfg["rlen"]], lengths[:n]
    return codes, lengths


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def lib_sha():
    import paper_1403_1706_b200 as qgm
    return qgm.build_stamp()  # sources + flags (nvcc output is not byte-reproducible)


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML in a background thread
    during the timed region (in-process NVML: no nvidia-smi subprocess)."""

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


def bind_to_gpu_numa(device):
    """Run this rank on the host cores NVML reports as local to its GPU (pinned
    buffers on the GPU's NUMA node). Returns the core count or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = int(vis.split(",")[device]) if vis and vis.split(",")[0].isdigit() else device
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


# ------------------------------------------------------------------ roofline
def algorithmic_bytes(kernel, cfg, st, n_reads):
    """Algorithmic HBM bytes of one launch of `kernel` on a batch with map stats
    `st` (DESIGN.md section 4 / SURVEY.md section 8(d)); None = not HBM-bound
    or no formula."""
    q, rlen = cfg["q"], cfg["rlen"]
    groups = (4 ** q) // 32
    V = st["index_occurrences"]
    text = n_reads * rlen / 4 + 4 * n_reads  # 2-bit reads + lengths
    if kernel == "k_filter":
        n_look = 2 * (cfg["ref_bp"] - q + 1)
        return cfg["ref_bp"] / 4 + 4 * n_look + 12 * st["lookups_hit"] + 4 * st["occurrences"] + 8 * st["raw_candidates"]
    if kernel == "k_join":
        # read join items (8 B) + occupancy words (4 B) and u16 group starts
        # (2 B) of the canonical index once + two S' entries per lookup hit +
        # one O word per occurrence visited + 8 B per candidate key written
        return 8 * V + 6 * groups + 8 * st["lookups_hit"] + 4 * st["occurrences"] + 8 * st["raw_candidates"]
    if kernel == "k_part_hist":
        return text
    if kernel == "k_part_scatter":
        return text + 8 * V
    if kernel == "k_refine_scatter":
        return 16 * V
    if kernel == "k_hash_insert":
        # timed only when the dedup ran on the whole candidate set (the 1/64
        # sample of the skip decision is timed as k_hash_insert_sample)
        return 8 * st["raw_candidates"] + 8 * st["unique_candidates"]
    if kernel == "k_strata_seg":
        return 16 * st["validated"] + 4 * n_reads + 16 * st["hits"]
    return None


VALIDATE_OPS_PER_ROW = 20  # int32 ops per banded Myers row (one band word)


def validate_ops(cfg, st):
    """SURVEY 8(d) algorithmic INT32 ops of the validation of one batch."""
    words = (cfg["band"] + 31) // 32
    return VALIDATE_OPS_PER_ROW * (cfg["rlen"] + cfg["band"] - 1) * words * st["unique_candidates"]


def load_ncu(config, sha):
    """ncu DRAM bytes / instruction counts per kernel captured from a build of
    these exact sources (tools/ncu_capture.py writes
    profiles/<round>/ncu_<config>.json with the library's build stamp); {}
    when absent or stale."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_{config}.json")), reverse=True):
        d = json.load(open(p))
        if d.get("lib_sha") == sha:
            d["_path"] = os.path.relpath(p, ROOT)
            return d
    return {}


# ------------------------------------------------------------------ GPU arm
def init_dist(args):
    """(rank, world, device index, dist or None, backend, oversubscribed)."""
    import torch
    from paper_1403_1706_b200 import sharding

    rank, world, local = sharding.world()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    n_dev = torch.cuda.device_count()
    if n_dev == 0:
        raise SystemExit("bench.py: no CUDA device (the product has no CPU path)")
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    oversub = local_world > n_dev
    device = local % n_dev
    torch.cuda.set_device(device)
    if world == 1:
        return rank, world, device, None, None, False
    import torch.distributed as dist
    backend = "gloo" if oversub else "nccl"
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", device))
    else:
        dist.init_process_group("gloo")
    return rank, world, device, dist, backend, oversub


def run_gpu(args):
    import ctypes as C

    import torch

    import paper_1403_1706_b200 as qgm
    from paper_1403_1706_b200 import sharding

    rank, world, device, dist, backend, oversub = init_dist(args)
    coll_dev = f"cuda:{device}" if backend == "nccl" else "cpu"
    numa_cores = None if oversub else bind_to_gpu_numa(device)
    cfg = CONFIGS[args.config]
    q, mode, band, rlen = cfg["q"], cfg["mode"], cfg["band"], cfg["rlen"]
    t_in = time.perf_counter()
    ref, cb = make_reference(qgm, cfg)
    blocks = sharding.read_blocks(rank, world, cfg["reads"] // cfg["batch"],
                                  cfg["reads"] // cfg["batch"] if cfg["strong"] else None)
    batches = [make_block(qgm, cfg, ref, cb, b) for b in blocks]
    inputs_s = time.perf_counter() - t_in
    n_rank_reads = sum(l.size for _, l in batches)
    stream = torch.cuda.Stream(device)
    ctx = qgm.Context(device, stream=stream.cuda_stream)
    # the reference: one H2D on rank 0, broadcast to the other ranks' devices
    ref_words = qgm.pack_codes(ref) if rank == 0 else None
    n_words = (cfg["ref_bp"] + 31) // 32 + 1
    d_ref, bcast_s = sharding.broadcast_reference(ref_words, n_words, dist, f"cuda:{device}")
    R = qgm.Reference(ctx, d_ref.data_ptr(), cb)
    del d_ref
    t0 = time.perf_counter()
    if cfg["mask_threshold"]:
        R.mask_repeats(q, cfg["mask_threshold"])
    R.prepare(q)  # reference preprocessing, once per reference and q, outside every timed region
    ref_prepare_s = time.perf_counter() - t0
    params = qgm.make_params(q=q, mode=mode, band_width=band, pct_identity=cfg["pct"])
    other = qgm.make_params(q=q, mode=1 - mode, band_width=band, pct_identity=cfg["pct"])
    lib = ctx.lib

    words = [qgm.pack_read_codes(c, rlen) for c, _ in batches]
    d_words = [torch.from_numpy(w.view(np.int64)).to(f"cuda:{device}") for w in words]
    d_len = [torch.from_numpy(l.view(np.int32)).to(f"cuda:{device}") for _, l in batches]
    # pinned host buffers for e2e, allocated before anything else large. The
    # streamed API takes one dense 2-bit stream per batch (2 bits per base, no
    # per-read padding) and, all reads being rlen long, no length array.
    uniform = all(bool(np.all(l == rlen)) for _, l in batches)
    h_dense = [torch.from_numpy(qgm.pack_codes(c).view(np.int64)).pin_memory() for c, _ in batches]
    h_len = [torch.from_numpy(l.view(np.int32)).pin_memory() for _, l in batches]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{device}")

    def map_batch(i, p=params, keep=False):
        rd = C.c_void_p()
        ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(d_words[i].data_ptr()), C.c_void_p(d_len[i].data_ptr()),
                                             batches[i][1].size, rlen, C.byref(rd)))
        h = C.c_void_p()
        try:
            ctx._check(lib.qgm_map(ctx.h, rd, R.h, C.byref(p), C.byref(h)))
            st = qgm.MapStats()
            lib.qgm_hits_stats(h, C.byref(st))
            out = {f: getattr(st, f) for f, _ in qgm.MapStats._fields_}
            if keep:
                hits = np.zeros(st.hits, qgm.HIT_DTYPE)
                ctx._check(lib.qgm_hits_download(ctx.h, h, qgm._ptr(hits)))
                out["_hits"] = hits
            return out
        finally:
            lib.qgm_hits_destroy(h)
            lib.qgm_reads_destroy(rd)

    def step_device(p=params):
        agg = None
        for i in range(len(batches)):
            st = map_batch(i, p)
            agg = st if agg is None else {k: agg[k] + st[k] for k in agg}
        return agg

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, K):
        times, out, launches = [], None, 0
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

    # ---------------- value: reads resident in HBM
    for _ in range(args.warmup):
        step_device()
    barrier()
    with ClockSampler(device, period=args.clock_period) as clk:
        times, st, launches = timed(step_device, args.steps)
        barrier()
    clocks = clk.summary()
    dev_ms = sum(times)

    # ---------------- the other mode on the same reads (BASELINE: best & all)
    for _ in range(max(1, args.warmup // 2)):
        step_device(other)
    barrier()
    otimes, ost, _ = timed(lambda: step_device(other), args.steps)
    other_ms = sum(otimes)

    # ---------------- e2e: host buffers through the C ABI, + end-of-run gather
    cap = max(int(max(st["hits"], ost["hits"]) / len(batches) * 1.25) + 4096, 1 << 16)
    n_e2e = args.steps * len(batches)
    h_hits = [torch.empty(cap * 16, dtype=torch.uint8).pin_memory() for _ in range(min(n_e2e, 2 * len(batches)))]
    gather = sharding.HostGather(dist, coll_dev)

    def run_batches(K):
        arr = (qgm.Batch * K)()
        for j in range(K):
            i = j % len(batches)
            arr[j] = qgm.Batch(h_dense[i].data_ptr(), None if uniform else h_len[i].data_ptr(), batches[i][1].size,
                               rlen, h_hits[j % len(h_hits)].data_ptr(), cap, 0, qgm.MapStats(), qgm.READS_DENSE, 0)
        ctx._check(lib.qgm_map_host_batches(ctx.h, arr, K, R.h, C.byref(params)))
        return arr

    def e2e_run(K):
        arr = run_batches(K)
        if world == 1:
            return arr, None
        # end-of-run gather: the last step's hits of every rank, straight from
        # the pinned hit buffers into the shared host buffer (batch order)
        views = [h_hits[j % len(h_hits)].numpy()[: arr[j].n_out * 16].view(qgm.HIT_DTYPE)
                 for j in range(K - len(batches), K)]
        return arr, gather.gather(views, qgm.HIT_DTYPE)

    e2e_run(max(args.steps, args.warmup, 3) * len(batches))  # warm-up with the timed batch count
    barrier()
    e2e_runs, gathered = [], None
    for _ in range(3):
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        arr, gathered = e2e_run(n_e2e)
        e1.record(stream)
        e1.synchronize()
        host_ms = (time.perf_counter() - t0) * 1e3
        # the gather is host-side after the stream drained: the larger of the
        # device interval and the host wall clock of the whole call
        e2e_runs.append(max(e0.elapsed_time(e1), host_ms))
    if gathered is not None:  # rank 0: batch-local read ids -> job read ids (outside the timing)
        blocks_of = [sharding.read_blocks(r, world, cfg["reads"] // cfg["batch"],
                                          cfg["reads"] // cfg["batch"] if cfg["strong"] else None)
                     for r in range(world)]
        seg = [b for r in range(world) for b in blocks_of[r]]
        counts = gather.last["segments"]
        base = np.repeat(np.array(seg, np.uint64) * cfg["batch"], counts).astype(np.uint32)
        gathered["read_id"] += base
    e2e_ms = sorted(e2e_runs)[1]
    e2e_hits_per_step = sum(arr[j].n_out for j in range(n_e2e)) / args.steps

    # ---------------- profile pass (per-kernel CUDA events; not part of `value`)
    ctx.profile(True)
    ctx.kernel_times(reset=True)
    ctx.stage_times(reset=True)
    prof_steps = max(1, min(3, args.steps))
    ptimes, _, _ = timed(step_device, prof_steps)
    ktimes = ctx.kernel_times(reset=True)
    stimes = ctx.stage_times(reset=True, host=True)
    ctx.profile(False)
    post = postprocess_pass(ctx, lib, C, qgm, R, d_words[0], d_len[0], batches[0][1].size, rlen, params, band)
    ibuild = index_build_pass(ctx, lib, C, qgm, stream, d_words[0], d_len[0], batches[0][1].size, rlen, q,
                              load_peaks()[0])

    # ---------------- parity sample: rank 0's first batch, downloaded
    first = map_batch(0, keep=True) if rank == 0 else None
    dev_ms, e2e_ms, other_ms = sharding.max_over_ranks([dev_ms, e2e_ms, other_ms], dist, device=coll_dev)
    job_reads = n_rank_reads if dist is None else int(sharding.sum_over_ranks([n_rank_reads], dist, coll_dev)[0])
    value = job_reads * args.steps / (dev_ms / 1e3)
    e2e_value = job_reads * args.steps / (e2e_ms / 1e3)
    other_value = job_reads * args.steps / (other_ms / 1e3)

    peak, peak_kind = load_peaks()
    sha = lib_sha()
    ncu = load_ncu(args.config, sha)
    bpl = len(batches)  # launches per step of every per-batch kernel
    per_launch = {k: v[0] / v[1] for k, v in ktimes.items()}
    st_batch = {k: v / bpl for k, v in st.items()}  # one batch's counts
    dom = max(per_launch, key=per_launch.get) if per_launch else None
    roof = None
    if dom:
        ab = algorithmic_bytes(dom, cfg, st_batch, cfg["batch"])
        traffic = ncu.get("kernels", {}).get(dom, {}).get("dram_bytes")
        if ab is not None:
            ach = ab / (per_launch[dom] / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": traffic, "peak_source": peak_kind,
                    "algorithmic_bytes": int(ab), "launch_ms": round(per_launch[dom], 4),
                    "share_of_step": round(ktimes[dom][0] / prof_steps / (sum(ptimes) / len(ptimes)), 4),
                    "traffic_source": ncu.get("_path") if traffic else "no ncu capture of this library build"}
    stage_roof = {}
    for kname, ms in per_launch.items():
        ab = algorithmic_bytes(kname, cfg, st_batch, cfg["batch"])
        if ab is not None:
            ach = ab / (ms / 1e3) / 1e9
            stage_roof[kname] = {"bound": "hbm", "achieved_gbs": round(ach, 1), "frac": round(ach / peak, 4),
                                 "ms": round(ms, 4)}
    if "k_validate" in per_launch:
        # INT-ALU bound: SURVEY 8(d) algorithmic ops against 148 SMs x 128
        # INT32 lanes x clock; the issue rate from ncu when captured
        clk_hz = (clocks.get("sm_mhz") or 1965) * 1e6
        ops = validate_ops(cfg, st_batch)
        peak_ops = 148 * 128 * clk_hz
        ach = ops / (per_launch["k_validate"] / 1e3)
        ent = {"bound": "INT32 ALU", "achieved_tops": round(ach / 1e12, 2), "peak_tops": round(peak_ops / 1e12, 2),
               "frac": round(ach / peak_ops, 4), "ms": round(per_launch["k_validate"], 4),
               "ops_formula": f"{VALIDATE_OPS_PER_ROW} x (n + B - 1) x ceil(B/32) x unique candidates"}
        inst = ncu.get("kernels", {}).get("k_validate", {}).get("warp_inst")
        if inst:
            ent["issue_frac"] = round(inst / (per_launch["k_validate"] / 1e3) / (148 * 4 * clk_hz), 4)
        stage_roof["k_validate"] = ent
        if dom == "k_validate":  # validation dominates (C3, C4, q=12): its INT-ALU roofline is the line's
            roof = {"bound": "int32 alu", "kernel": "k_validate", "achieved": ent["achieved_tops"],
                    "peak": ent["peak_tops"], "unit": "TOP/s", "frac": ent["frac"],
                    "traffic": ncu.get("kernels", {}).get("k_validate", {}).get("dram_bytes"),
                    "peak_source": "148 SMs x 128 INT32 lanes x measured SM clock",
                    "ops_formula": ent["ops_formula"], "launch_ms": ent["ms"],
                    "share_of_step": round(ktimes["k_validate"][0] / prof_steps / (sum(ptimes) / len(ptimes)), 4),
                    "traffic_source": ncu.get("_path") if ncu else "no ncu capture of this library build"}
    step_mean = sum(ptimes) / len(ptimes)
    f_filt = (stimes.get("filter", 0.0) / prof_steps) / step_mean if step_mean else None

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "reads/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "strong" if cfg["strong"] else "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded reference and simulated reads)",
        "config": config_dict(args.config, cfg, world),
        "mode_value": {MODES[mode]: round(value, 1), MODES[1 - mode]: round(other_value, 1)},
        MODES[1 - mode].replace("-stratum", "") + "_mode": {
            "value": round(other_value, 1), "ms_per_step": round(other_ms / args.steps, 3),
            "hits_per_step": int(ost["hits"]), "note": "same reads, device-resident, other strata mode"},
        "e2e": {"value": round(e2e_value, 1), "unit": "reads/s", "ms_per_step": round(e2e_ms / args.steps, 3),
                "h2d_bytes_per_step": int(sum(t.numel() * 8 for t in h_dense)
                                          + (0 if uniform else sum(l.nbytes for _, l in batches))),
                "d2h_bytes_per_step": int(e2e_hits_per_step * 16),
                "api": "qgm_map_host_batches (streamed; copies overlap mapping; dense 2-bit reads)"
                       + (" + end-of-run HostGather" if world > 1 else ""),
                "gather": {k: v for k, v in gather.last.items() if k != "counts"},
                "runs": 3, "statistic": "median of 3 timed runs of K steps"},
        "gpu_launches": int(launches),
        "roofline": roof,
        "stage_roofline": stage_roof,
        "f_filt": round(f_filt, 4) if f_filt is not None else None,
        "clocks": clocks,
        "step_ms": [round(t, 3) for t in times],
        "e2e_step_ms": [round(t / args.steps, 3) for t in e2e_runs],
        "stages_ms_per_step": {k: round(v / prof_steps, 4) for k, v in stimes.items() if v},
        "kernels_ms_per_launch": {k: round(v, 4) for k, v in per_launch.items()},
        "counts": st,
        "lib_sha": sha,
        "reference_prepare_s": round(ref_prepare_s, 3),
        "reference_distribution": {"method": "H2D on rank 0 + broadcast" if world > 1 else "H2D",
                                   "backend": backend, "seconds": round(bcast_s, 3)},
        "inputs_s": round(inputs_s, 2),
        "host_binding": {"cores": numa_cores, "rule": "NVML CPU affinity of the rank's GPU"},
        "postprocess": post,
        "index_build": ibuild,
    }
    if world > 1:
        line["backend"] = backend
        line["oversubscribed"] = oversub
        if oversub:
            line["note"] = (f"{world} ranks share {torch.cuda.device_count()} GPU(s) over gloo: functional "
                            "multi-rank run, not a scaling measurement")
        if rank == 0 and gathered is not None:
            line["gathered"] = {"hits": int(gathered.size), "digest": sharding.hits_digest(gathered)}
    if rank == 0:
        line["parity"] = None
        if world == 1 and (not args.no_cpu or args.check != "off") or (world > 1 and args.check != "off"):
            leg = cpu_leg_subprocess(args, first["_hits"], want_baseline=(world == 1 and not args.no_cpu))
            if leg.get("cpu_baseline"):
                line["cpu_baseline"] = leg["cpu_baseline"]
            line["parity"] = leg.get("parity")
        print(json.dumps(line), flush=True)
    del R
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_refshard(args):
    """--shard ref: every rank maps the SAME read batch
    against its share of the reference (refshard.plan: equal owned lengths,
    chromosomes cut where a share fills); the hit records stay on the device
    and the exchange -- MIN all-reduce of each read's best k (best mode) and an
    all-to-all of the records to the read's owner -- runs on CUDA tensors over
    NCCL (gloo + host tensors when ranks share a GPU). One step = one batch
    mapped by the whole job; timed on the host around the synchronised step
    (the exchange is host-driven), max over ranks."""
    import ctypes as C

    import torch

    import paper_1403_1706_b200 as qgm
    from paper_1403_1706_b200 import refshard, sharding

    rank, world, device, dist, backend, oversub = init_dist(args)
    xdev = "cpu" if backend == "gloo" else f"cuda:{device}"
    coll_dev = xdev
    cfg = CONFIGS[args.config]
    q, mode, band, rlen = cfg["q"], cfg["mode"], cfg["band"], cfg["rlen"]
    ref, cb = make_reference(qgm, cfg)
    codes, lengths = make_block(qgm, cfg, ref, cb, 0)
    ctx = qgm.Context(device)
    mask = None
    if cfg["mask_threshold"]:  # counted over whole chromosomes, then sliced per piece
        Rw = qgm.Reference.from_codes(ctx, ref, cb).mask_repeats(q, cfg["mask_threshold"])
        mask = Rw.mask()
        Rw.close()
    mine = refshard.plan(cb, world, rlen, band)[rank]
    pc, pcb, pm = refshard.piece_reference(ref, cb, mine, mask)
    t0 = time.perf_counter()
    R = qgm.Reference.from_codes(ctx, pc, pcb, mask=pm).prepare(q) if mine else None
    prep_s = time.perf_counter() - t0
    words = qgm.pack_read_codes(codes, rlen)
    d_words = torch.from_numpy(words.view(np.int64)).to(f"cuda:{device}")
    d_len = torch.from_numpy(lengths.view(np.int32)).to(f"cuda:{device}")
    pall = qgm.make_params(q=q, mode=1, band_width=band, pct_identity=cfg["pct"])
    lib = ctx.lib
    n_reads = lengths.size

    def step():
        t_map = time.perf_counter()
        local = torch.zeros((0, 4), dtype=torch.int32, device=xdev)
        st = None
        if R is not None:
            rd, h = C.c_void_p(), C.c_void_p()
            ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(d_words.data_ptr()), C.c_void_p(d_len.data_ptr()),
                                                 n_reads, rlen, C.byref(rd)))
            try:
                ctx._check(lib.qgm_map(ctx.h, rd, R.h, C.byref(pall), C.byref(h)))
                n = C.c_uint64()
                lib.qgm_hits_count(h, C.byref(n))
                s_ = qgm.MapStats()
                lib.qgm_hits_stats(h, C.byref(s_))
                st = {f: getattr(s_, f) for f, _ in qgm.MapStats._fields_}
                local = torch.empty((n.value, 4), dtype=torch.int32, device=f"cuda:{device}")
                if n.value:
                    ctx._check(lib.qgm_hits_download(ctx.h, h, C.c_void_p(local.data_ptr())))
            finally:
                lib.qgm_hits_destroy(h)
                lib.qgm_reads_destroy(rd)
            local = refshard.own_and_translate(local.to(xdev), mine)
        if xdev.startswith("cuda"):
            torch.cuda.synchronize(device)
        t_x = time.perf_counter()
        out = refshard.combine(local, n_reads, mode, dist)
        if xdev.startswith("cuda"):
            torch.cuda.synchronize(device)
        t_end = time.perf_counter()
        return out, st, (t_x - t_map) * 1e3, (t_end - t_x) * 1e3

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    barrier()
    times, xms, mms = [], [], []
    with ClockSampler(device, period=args.clock_period) as clk:
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            out, st, m_ms, x_ms = step()
            times.append((time.perf_counter() - t0) * 1e3)
            mms.append(m_ms)
            xms.append(x_ms)
    clocks = clk.summary()
    tot, xsum, msum = sharding.max_over_ranks([sum(times), sum(xms), sum(mms)], dist, device=coll_dev)
    mine_hits = refshard.from_records(out)
    gathered = sharding.HostGather(dist, coll_dev).gather(mine_hits)
    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": round(n_reads * args.steps / (tot / 1e3), 1), "unit": "reads/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic (seeded reference and simulated reads)", "shard": "reference",
                "config": dict(config_dict(args.config, cfg, world), reads_per_step=n_reads,
                               parallelism=f"reference sharded over {world} rank(s), reads replicated"),
                "map_ms_per_step": round(msum / args.steps, 3), "exchange_ms_per_step": round(xsum / args.steps, 3),
                "exchange": {"backend": backend or "none (world 1)", "device": xdev,
                             "steps": "MIN all-reduce of per-read k (best mode) + all-to-all of 16-byte records"},
                "piece_prepare_s": round(prep_s, 3), "clocks": clocks, "counts_rank0": st,
                "hits": int(gathered.size), "digest": sharding.hits_digest(gathered)}
        if oversub:
            line["oversubscribed"] = True
        if args.check != "off":  # whole reference on rank 0's GPU: same hits?
            Rw = qgm.Reference.from_codes(ctx, ref, cb, mask=mask)
            reads = qgm.Reads(ctx, words, lengths, rlen)
            want, _ = ctx.map(reads, Rw, q=q, mode=mode, band_width=band, pct_identity=cfg["pct"])
            line["parity"] = {"ok": sharding.hits_digest(want) == line["digest"], "whole_reference_hits": int(want.size),
                              "what": "digest of the gathered per-owner hits vs one GPU mapping the whole reference"}
            reads.close()
            Rw.close()
        print(json.dumps(line), flush=True)
    if R is not None:
        R.close()
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def postprocess_pass(ctx, lib, C, qgm, R, d_words, d_len, n_reads, rlen, params, band):
    """SPEC.md:446-483 tail on one batch's device-resident hits (not part of
    `value`): hit_rank and traceback_cigar, CUDA-event kernel times, second of
    two runs."""
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
        max_ops = 2 * band + 16
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


def index_build_pass(ctx, lib, C, qgm, stream, d_words, d_len, n_reads, rlen, q, peak):
    """build_qgroup_index<u32> (qgroup_index.hpp:124-180) of one batch through
    the API (qgm_index_build: the full four-array read index of Alg. 1, not
    used by the map path), CUDA events on the library stream, median of 3 after
    a warm-up; algorithmic bytes N*n/4 (2-bit reads) + 8*Gq (I and S) +
    4*(D+1) (S') + 4*V (O)."""
    import torch
    rd = C.c_void_p()
    ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(d_words.data_ptr()), C.c_void_p(d_len.data_ptr()),
                                         n_reads, rlen, C.byref(rd)))
    try:
        times, info = [], None
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h = C.c_void_p()
            ctx._check(lib.qgm_index_build(ctx.h, rd, q, 32, 0, C.byref(h)))
            e1.record(stream)
            e1.synchronize()
            info = qgm.IndexInfo()
            ctx._check(lib.qgm_index_info_get(h, C.byref(info)))
            lib.qgm_index_destroy(h)
            if it:
                times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        ab = n_reads * rlen / 4 + 8 * info.group_count + 4 * (info.distinct + 1) + 4 * info.occurrences
        return {"api": "qgm_index_build (build_qgroup_index<uint32_t>, not sampled)", "q": q, "ms": round(ms, 4),
                "groups": info.group_count, "distinct": info.distinct, "occurrences": info.occurrences,
                "algorithmic_bytes": int(ab), "achieved_gbs": round(ab / (ms / 1e3) / 1e9, 1),
                "frac": round(ab / (ms / 1e3) / 1e9 / peak, 4)}
    finally:
        lib.qgm_reads_destroy(rd)


# ------------------------------------------------------------------ CPU legs
def cpu_leg_subprocess(args, gpu_hits, want_baseline):
    """Runs `bench.py --cpu-leg` in a child process (the GPU process never maps
    oracle/ code) on rank 0's first batch: timing (cpu_baseline) and the
    parity digest against the GPU hits of the same reads."""
    cfg = CONFIGS[args.config]
    sample = cfg["batch"] if args.check == "full" else min(cfg["cpu_sample"], cfg["batch"])
    with tempfile.TemporaryDirectory() as td:
        gp = os.path.join(td, "gpu_hits.npy")
        np.save(gp, gpu_hits[gpu_hits["read_id"] < sample])
        out = os.path.join(td, "leg.json")
        cmd = [sys.executable, os.path.abspath(__file__), "--cpu-leg", "--config", args.config,
               "--sample", str(sample), "--gpu-hits", gp, "--leg-out", out,
               "--cpu-samples", str(args.cpu_samples if want_baseline else 1)]
        env = dict(os.environ)
        env.pop("CUDA_VISIBLE_DEVICES", None)
        r = subprocess.run(cmd, capture_output=True, text=True, env=env)
        if r.returncode != 0 or not os.path.exists(out):
            return {"parity": {"ok": None, "error": (r.stderr or r.stdout)[-800:]}}
        leg = json.load(open(out))
    if not want_baseline:
        leg.pop("cpu_baseline", None)
    return leg


def cpu_map(cfg, ref, cb, codes, lengths, threads, samples=1):
    """The CPU path: the reference's build_qgroup_index (oracle/_ref, compiled
    from /root/reference) + the restated stages 2-5; the oracle port when the
    reference shim is absent. Best of `samples` runs."""
    from oracle.pyoracle import REF_SO, Oracle, RefShim, repeat_mask
    kind = "reference" if os.path.exists(REF_SO) else "port"
    impl = RefShim() if kind == "reference" else Oracle()
    mask = repeat_mask(ref, cb, cfg["q"], cfg["mask_threshold"]) if cfg["mask_threshold"] else None
    best, hits, st = None, None, None
    for _ in range(samples):
        t0 = time.perf_counter()
        hits, st = impl.map(ref, cb, codes, cfg["rlen"], lengths, q=cfg["q"], mode=cfg["mode"], band=cfg["band"],
                            pct=cfg["pct"], threads=threads, mask=mask)
        dt = time.perf_counter() - t0
        if best is None or dt < best[0]:
            best = (dt, st)
    return kind, best[0], hits, best[1]


def run_gen_inputs(args):
    """--gen-inputs PATH (child process): the config's reference and the
    first `sample` reads of block 0, written to PATH (npz) -- so the CPU
    processes (reference arm, CPU leg) never map the repo's synthetic-data
    library, only numpy arrays and the reference / oracle code."""
    import paper_1403_1706_b200 as qgm
    cfg = CONFIGS[args.config]
    ref, cb = make_reference(qgm, cfg)
    codes, lengths = make_block(qgm, cfg, ref, cb, 0, args.sample or None)
    np.savez(args.gen_inputs, ref=ref, cb=cb, codes=codes, lengths=lengths)


def isolated_inputs(config, sample):
    """(ref, chrom_begin, codes, lengths) generated in a child process."""
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "inputs.npz")
        subprocess.run([sys.executable, os.path.abspath(__file__), "--config", config, "--gen-inputs", path,
                        "--sample", str(sample)], check=True)
        z = np.load(path)
        return z["ref"], z["cb"], z["codes"], z["lengths"]


def run_cpu_leg(args):
    """--cpu-leg (child of the GPU arm): the CPU path on the first `sample`
    reads of block 0 of rank 0, timed, compared with the GPU hits."""
    from paper_1403_1706_b200 import sharding
    cfg = CONFIGS[args.config]
    ref, cb, codes, lengths = isolated_inputs(args.config, args.sample)
    threads = os.cpu_count() or 1
    kind, sec, hits, st = cpu_map(cfg, ref, cb, codes, lengths, threads, samples=args.cpu_samples)
    res = {"cpu_baseline": {
        "value": round(args.sample / sec, 1), "unit": "reads/s", "cores": threads, "kind": kind,
        "cpu": cpu_info(),
        "sample": f"first {args.sample} reads of the config's first {cfg['batch']}-read batch vs the full "
                  f"{cfg['ref_bp']} bp reference; index = reference build_qgroup_index (qgroup_index.hpp:124-180), "
                  f"stages 2-5 = oracle restatement; best of {args.cpu_samples}, {sec:.2f} s",
        "stage_seconds": st.get("stage_seconds"),
        "counts": {k: v for k, v in st.items() if k != "stage_seconds"}}}
    if args.gpu_hits:
        g = np.load(args.gpu_hits)
        gd, cd = sharding.hits_digest(g), sharding.hits_digest(hits)
        res["parity"] = {"ok": gd == cd, "reads": args.sample, "gpu_hits": int(g.size), "cpu_hits": int(hits.size),
                         "gpu_digest": gd, "cpu_digest": cd,
                         "what": "sha256 of the sorted (read, chrom, ref_start, strand, edits) hit set of the "
                                 "sampled reads, GPU (full batch, restricted to them) vs CPU path"}
    json.dump(res, open(args.leg_out, "w"))


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores (rank 0
    only), each step a bounded sample of the config's first batch."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    sample = min(cfg["cpu_sample"], cfg["batch"])
    ref, cb, codes, lengths = isolated_inputs(args.config, sample)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_map(cfg, ref, cb, codes, lengths, threads)
    times, st, kind = [], None, None
    for _ in range(args.steps):
        kind, sec, hits, st = cpu_map(cfg, ref, cb, codes, lengths, threads)
        times.append(sec)
    total = sum(times)
    value = sample * args.steps / total
    line = {"metric": METRIC, "value": round(value, 1), "unit": "reads/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 1),
            "higher_is_better": True, "scaling": "strong" if cfg["strong"] else "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seeded reference and simulated reads)", "impl": "reference",
            "config": config_dict(args.config, cfg, world),
            "cpu_baseline": {"value": round(value, 1), "unit": "reads/s", "cores": threads, "kind": kind,
                             "cpu": cpu_info(),
                             "sample": f"each step: the first {sample} reads of the config's first batch vs the "
                                       f"full {cfg['ref_bp']} bp reference; index = reference build_qgroup_index "
                                       f"(qgroup_index.hpp:124-180), stages 2-5 = oracle restatement",
                             "stage_seconds_last_step": st.get("stage_seconds")},
            "e2e": {"value": round(value, 1), "unit": "reads/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "counts": {k: v for k, v in st.items() if k != "stage_seconds"}}
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args):
    """`--gpus N` without a torchrun environment: one process per GPU."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.run(cmd).returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--check", default=None, choices=["off", "sample", "full"],
                    help="parity of rank 0's first batch vs the CPU path (subprocess); default: sample at N = 1, "
                         "off at N > 1 (the gathered digest is reported there)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (parity still per --check)")
    ap.add_argument("--cpu-samples", type=int, default=1, help="cpu_baseline: best of this many runs")
    ap.add_argument("--clock-period", type=float, default=0.005, help="NVML clock sampling period (s)")
    ap.add_argument("--shard", default="reads", choices=["reads", "ref"],
                    help="reads: read-sharded replicas (default); ref: reference sharded, reads replicated, "
                         "device-resident exchange (SURVEY 8(f) row 2)")
    # internal: the CPU leg child process
    ap.add_argument("--cpu-leg", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--sample", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--gpu-hits", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--leg-out", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--gen-inputs", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gen_inputs:
        return run_gen_inputs(args)
    if args.cpu_leg:
        return run_cpu_leg(args)
    if args.check is None:
        args.check = "sample" if args.gpus == 1 else "off"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.shard == "ref":
        return run_refshard(args)
    return run_gpu(args)


if __name__ == "__main__":
    main()

"""GPU parity tests through the C ABI (libqgm_b200.so) against the CPU oracle.

* the C++ parity suites in tests/cpp (Catch2-style, reading like the
  reference's own tests) -- one pytest case per binary;
* config C1 at full size (1 Mbp random reference, 10k simulated 100 bp reads
  at 3% edits, q=12, best-stratum) through the python binding, hit-for-hit
  against the oracle, plus all-mode and q=16 variants;
* size-independent properties at the bench size (C2 shape): e2e host entry ==
  device entry, best-stratum subset of all, truth recall.
"""
import os
import subprocess

import numpy as np
import pytest

from qgm_testutil import ROOT

pytestmark = pytest.mark.gpu

CPP = ["test_qgroup_index", "test_filter", "test_validate", "test_map", "test_pipeline"]


@pytest.mark.parametrize("name", CPP)
def test_cpp_parity_suite(name):
    exe = os.path.join(ROOT, "tests", "cpp", "build", name)
    assert os.path.exists(exe), f"{exe} not built (make tests)"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=1800)
    tail = out.stdout[-3000:] + "\n" + out.stderr[-3000:]
    assert out.returncode == 0, tail
    assert " 0 failed" in out.stdout.strip().splitlines()[-1], tail


def _c1(qgm, n_reads=10_000, L=1_000_000, err=0.03, seed=1):
    ref = qgm.random_reference(seed, L)
    cb = np.array([0, L], np.uint64)
    codes, lengths, tc, tp, ts = qgm.simulate_reads(seed + 1, ref, cb, n_reads, 100, err)
    return ref, cb, codes, lengths, tp, ts


def _validated_agrees(st, ost, mode, info=None):
    """The `validated` statistic (kept candidates before the strata) equals
    the oracle's in both modes: validation abandons a candidate only once its
    lower bound exceeds the identity threshold's k, never against the read's
    best k (mode is kept for the call sites)."""
    assert st["validated"] == ost["validated"], (st, ost, mode, info)


def _same(a, b):
    cols = ("read_id", "chrom", "ref_start", "edits", "strand")
    return a.size == b.size and all(np.array_equal(a[c], b[c]) for c in cols)


@pytest.mark.parametrize("mode,q", [(0, 12), (1, 12), (0, 16), (1, 16)])
def test_c1_full_size_matches_oracle(ctx, oracle, mode, q):
    import paper_1403_1706_b200 as qgm
    ref, cb, codes, lengths, tp, ts = _c1(qgm)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    got, st = ctx.map(reads, R, q=q, mode=mode)
    want, ost = oracle.map(ref, cb, codes, 100, lengths, q=q, mode=mode)
    assert st["unique_candidates"] == ost["unique_candidates"]
    _validated_agrees(st, ost, mode)
    assert _same(got, want), (got.size, want.size)
    # sensitivity sanity: most reads map at their true origin (3% edits, q=12)
    if q == 12 and mode == 0:
        mapped = np.zeros(lengths.size, bool)
        mapped[got["read_id"]] = True
        assert mapped.mean() > 0.97


@pytest.mark.parametrize("unpacked", [False, True])
def test_repetitive_reference_and_mask_match_oracle(ctx, oracle, monkeypatch, unpacked):
    """Repeats (long occurrence intervals, warp-cooperative expansion), two
    chromosomes, a repeat mask; both reference-index layouts (compare base
    packed into O, or the separate byte array used above 2^29 padded bases)."""
    import paper_1403_1706_b200 as qgm
    if unpacked:
        monkeypatch.setenv("QGM_REF_UNPACKED", "1")
    L = 300_000
    ref = qgm.repetitive_reference(5, L)
    cb = np.array([0, 100_000, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(6, ref, cb, 3000, 100, 0.03)
    # repeat mask: forward q-gram frequency per chromosome > 20
    q = 12
    mask = np.zeros(L, np.uint8)
    for c in range(2):
        seq = ref[cb[c]:cb[c + 1]]
        w = np.lib.stride_tricks.sliding_window_view(seq, q)
        codes_c = (w.astype(np.uint64) * (4 ** np.arange(q - 1, -1, -1, dtype=np.uint64))).sum(1)
        u, inv, cnt = np.unique(codes_c, return_inverse=True, return_counts=True)
        mask[cb[c]:cb[c] + w.shape[0]] = (cnt[inv] > 20)
    for m in (None, mask):
        R = qgm.Reference.from_codes(ctx, ref, cb, mask=m)
        reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
        got, st = ctx.map(reads, R, q=q, mode=1)
        want, ost = oracle.map(ref, cb, codes, 100, lengths, q=q, mode=1, mask=m)
        assert _same(got, want), (m is None, got.size, want.size)


@pytest.mark.parametrize("q,strands", [(12, 1), (12, 2), (16, 3), (16, 1)])
def test_repeat_intervals_skip_only_suppressed_occurrences(ctx, oracle, q, strands):
    """Tandem repeats give q-gram intervals of thousands of occurrences, where
    the join skips the (strand flag, compare base) classes the run-start rule
    suppresses (the reference intervals are sorted by that class): one strand
    or both, every hit and statistic identical to the oracle."""
    import paper_1403_1706_b200 as qgm
    L = 300_000
    ref = qgm.repetitive_reference(40 + q, L)
    cb = np.array([0, 170_000, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(41 + q, ref, cb, 3000, 100, 0.03)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    got, st = ctx.map(reads, R, q=q, mode=1, strands=strands)
    want, ost = oracle.map(ref, cb, codes, 100, lengths, q=q, mode=1, strands=strands)
    assert _same(got, want), (got.size, want.size)
    assert st["unique_candidates"] == ost["unique_candidates"], (st, ost)
    _validated_agrees(st, ost, 1)


@pytest.mark.parametrize("skewed", [False, True])
def test_read_index_build_wide_buckets_and_fallback(ctx, oracle, skewed):
    """qgm_index_build at q=16 takes 2^16-code buckets from the raw-code
    partition; a bucket with more distinct codes than the emit's shared
    counters hold (every read = AAAAAAAA + 8 random bases: ~58k distinct codes
    in bucket 0) falls back to 2^13-code buckets. Both equal the oracle's
    build_qgroup_index (positions normalised inside intervals)."""
    import paper_1403_1706_b200 as qgm
    rng = np.random.default_rng(7 + skewed)
    if skewed:
        n, stride = 150_000, 16
        codes = rng.integers(0, 4, n * stride).astype(np.uint8)
        codes.reshape(n, stride)[:, :8] = 0
    else:
        n, stride = 20_000, 100
        codes = rng.integers(0, 4, n * stride).astype(np.uint8)
    lengths = np.full(n, stride, np.uint32)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, stride)
    idx = qgm.Index.build(ctx, reads, 16).normalize()
    I, S, S1, O = idx.arrays()
    wI, wS, wS1, wO = oracle.build_index(codes, stride, lengths, 16)
    from oracle.pyoracle import sort_intervals
    assert np.array_equal(I, wI) and np.array_equal(S, wS) and np.array_equal(S1, wS1)
    assert np.array_equal(O, sort_intervals(wS1, wO))


def test_device_scan_matches_reference_semantics(ctx):
    import paper_1403_1706_b200 as qgm
    sums, tot = ctx.exclusive_scan(np.array([3, 0, 2], np.uint32))
    assert sums.tolist() == [0, 3, 3] and tot == 5
    v = np.random.default_rng(1).integers(0, 100, 1_000_003).astype(np.uint32)
    sums, tot = ctx.exclusive_scan(v)
    assert np.array_equal(sums, (np.cumsum(v, dtype=np.uint64) - v).astype(np.uint32))
    with pytest.raises(qgm.InputError):
        ctx.exclusive_scan(np.full(3, 0xF0000000, np.uint32))


@pytest.mark.parametrize("n", [1, 15, 16, 17, 1023, 10_001, 16_383, 16_384, 16_385, 65_537])
def test_device_scan_around_the_single_cta_tile(ctx, n):
    """The one-CTA register scan covers n <= 16384 (16 per thread, vector
    loads only for full runs); above it the three-kernel tiled scan."""
    v = np.random.default_rng(n).integers(0, 1 << 16, n).astype(np.uint32)
    sums, tot = ctx.exclusive_scan(v)
    ref = np.cumsum(v, dtype=np.uint64) - v
    assert np.array_equal(sums, ref.astype(np.uint32)) and tot == int(v.sum(dtype=np.uint64))


def test_c2_shape_properties(ctx):
    """Bench-size batch (1M reads against a 100 Mbp reference, q=16): the e2e
    host entry point equals the device-resident one; best-stratum hits are a
    subset of all-mode hits; nearly every read maps at its true origin."""
    import paper_1403_1706_b200 as qgm
    L, N = 100_000_000, 1_000_000
    ref = qgm.random_reference(11, L)
    cb = np.array([0, L], np.uint64)
    codes, lengths, tc, tp, ts = qgm.simulate_reads(12, ref, cb, N, 100, 0.03)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    words = qgm.pack_read_codes(codes, 100)
    reads = qgm.Reads(ctx, words, lengths, 100)
    best, st = ctx.map(reads, R, q=16, mode=0)
    allm, _ = ctx.map(reads, R, q=16, mode=1)
    host, st2 = ctx.map_host(words, lengths, 100, R, q=16, mode=0)
    assert _same(best, host) and st == st2
    key = lambda h: set(zip(h["read_id"].tolist(), h["chrom"].tolist(), h["ref_start"].tolist(),
                            h["strand"].tolist()))
    assert key(best) <= key(allm)
    # truth: forward start of the fragment; the hit may start a few bases off
    # when the first bases carry edits, so test within +-8 bp.
    first = np.full(N, -1, np.int64)
    strand = np.zeros(N, np.uint8)
    first[best["read_id"][::-1]] = best["ref_start"][::-1].astype(np.int64)
    strand[best["read_id"][::-1]] = best["strand"][::-1]
    ok = (np.abs(first - tp.astype(np.int64)) <= 8) & (strand == ts)
    assert ok.mean() > 0.95, ok.mean()


def test_c3_shard_full_batch_matches_oracle_on_a_read_sample(ctx, oracle):
    """BASELINE config 3's per-GPU shard at full size (bench.py C3shard: 3.1
    Gbp in 24 chromosomes, q=16, best-stratum): the whole 1.25M-read batch
    mapped on the device -- the unpacked O layout above 2^28 padded bases,
    unstaged S'/O slices, the sampled dedup-skip decision -- and the hits of
    its first 20k reads identical to the CPU oracle on those reads (a read's
    hits depend only on the read and the reference)."""
    import bench
    import paper_1403_1706_b200 as qgm
    cfg = bench.CONFIGS["C3shard"]
    ref, cb = bench.make_reference(qgm, cfg)
    codes, lengths = bench.make_block(qgm, cfg, ref, cb, 0)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, cfg["rlen"])
    got, st = ctx.map(reads, R, q=16, mode=0)
    del reads, R
    assert st["hits"] > 0.99 * lengths.size
    S = 20_000
    want, _ = oracle.map(ref, cb, codes[: S * cfg["rlen"]], cfg["rlen"], lengths[:S], q=16, mode=0)
    assert _same(got[got["read_id"] < S], want), (int((got["read_id"] < S).sum()), want.size)


def test_c2_full_size_hit_parity_with_oracle(ctx, oracle):
    """The bench workload itself (100 Mbp, 1M reads, q=16, all-hits): every
    hit identical to the CPU oracle (Alg. 2 multiset + sort/unique + banded DP
    restatement + strata)."""
    import paper_1403_1706_b200 as qgm
    L, N = 100_000_000, 1_000_000
    ref = qgm.random_reference(7, L)
    cb = np.array([0, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(1000, ref, cb, N, 100, 0.03)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    got, st = ctx.map(reads, R, q=16, mode=1)
    want, ost = oracle.map(ref, cb, codes, 100, lengths, q=16, mode=1)
    assert st["unique_candidates"] == ost["unique_candidates"]
    assert _same(got, want), (got.size, want.size)


@pytest.mark.parametrize("stride,band", [(18, 32), (20, 32), (130, 32), (600, 64)])
def test_variable_length_reads_match_oracle(ctx, oracle, stride, band):
    """Reads of mixed lengths (some shorter than q, some filling the stride),
    several chromosomes, both modes: exercises the per-read length paths (the
    join item's n - q - o field, and -- for strides above q + 511 -- the
    join's reload of the read length). Strides 18 and 20 at q=12 leave 7 and 9
    q-gram slots per read: the partition's one-slot-per-thread path and its
    8-slot runs that cross a read boundary."""
    import paper_1403_1706_b200 as qgm
    L = 400_000
    ref = qgm.random_reference(21, L)
    cb = np.array([0, 150_000, 260_000, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(22, ref, cb, 2000, stride, 0.03)
    rng = np.random.default_rng(5)
    lengths = np.minimum(lengths, rng.integers(5, stride + 1, lengths.size).astype(np.uint32))
    lengths[:7] = stride
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, stride)
    for mode in (0, 1):
        got, st = ctx.map(reads, R, q=12, mode=mode, band_width=band)
        want, ost = oracle.map(ref, cb, codes, stride, lengths, q=12, mode=mode, band=band)
        assert st["unique_candidates"] == ost["unique_candidates"]
        assert _same(got, want), (mode, got.size, want.size)


def test_reads_with_many_hits_match_oracle(ctx, oracle):
    """A 300 bp unit repeated 60 times (with a few point differences per copy)
    between random flanks: reads from the unit have more than 32 hits each in
    all mode, which sends them through the strata stage's radix-sorted
    big-segment path; best-stratum keeps the exact-copy ties."""
    import paper_1403_1706_b200 as qgm
    rng = np.random.default_rng(9)
    unit = rng.integers(0, 4, 300).astype(np.uint8)
    copies = []
    for _ in range(60):
        u = unit.copy()
        pos = rng.integers(0, 300, 2)
        u[pos] = rng.integers(0, 4, 2)
        copies.append(u)
    ref = np.concatenate([qgm.random_reference(3, 50_000), *copies, qgm.random_reference(4, 50_000)]).astype(np.uint8)
    cb = np.array([0, ref.size], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(8, ref, cb, 1500, 100, 0.02)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    for mode in (1, 0):
        got, st = ctx.map(reads, R, q=12, mode=mode)
        want, ost = oracle.map(ref, cb, codes, 100, lengths, q=12, mode=mode)
        assert _same(got, want), (mode, got.size, want.size)
        if mode == 1:
            assert np.bincount(got["read_id"]).max() > 32


def test_device_repeat_mask_matches_numpy_and_maps_like_the_oracle(ctx, oracle):
    """qgm_ref_mask_repeats (per-chromosome forward q-gram
    frequency) equals a numpy count on a repetitive two-chromosome reference;
    the masked reference then maps exactly like the oracle given that mask."""
    import paper_1403_1706_b200 as qgm
    L = 300_000
    ref = qgm.repetitive_reference(15, L)
    cb = np.array([0, 120_000, L], np.uint64)
    q, thr = 12, 30
    want = np.zeros(L, np.uint8)
    for c in range(2):
        seq = ref[cb[c]:cb[c + 1]]
        w = np.lib.stride_tricks.sliding_window_view(seq, q)
        codes_c = (w.astype(np.uint64) * (4 ** np.arange(q - 1, -1, -1, dtype=np.uint64))).sum(1)
        u, inv, cnt = np.unique(codes_c, return_inverse=True, return_counts=True)
        want[cb[c]:cb[c] + w.shape[0]] = cnt[inv] > thr
    R = qgm.Reference.from_codes(ctx, ref, cb)
    R.mask_repeats(q, thr)
    got_mask = R.mask()
    assert want.sum() > 0 and np.array_equal(got_mask, want)
    codes, lengths, *_ = qgm.simulate_reads(16, ref, cb, 3000, 100, 0.03)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    got, st = ctx.map(reads, R, q=q, mode=1)
    exp, ost = oracle.map(ref, cb, codes, 100, lengths, q=q, mode=1, mask=want)
    assert _same(got, exp), (got.size, exp.size)


def test_streamed_batches_equal_single_calls(ctx):
    """qgm_map_host_batches (copies of batch i+1 / hits of batch i-1 overlap
    the mapping of batch i) returns, batch for batch, exactly what
    qgm_map_host returns; batches of different sizes and strides."""
    import paper_1403_1706_b200 as qgm
    L = 500_000
    ref = qgm.random_reference(31, L)
    cb = np.array([0, 200_000, L], np.uint64)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    batches = []
    for i, (n, stride) in enumerate([(3000, 100), (500, 150), (4000, 100), (1, 100), (2500, 120)]):
        codes, lengths, *_ = qgm.simulate_reads(40 + i, ref, cb, n, stride, 0.03)
        batches.append((qgm.pack_read_codes(codes, stride), lengths, stride))
    got = ctx.map_host_batches(batches, R, q=14, mode=1)
    for (words, lengths, stride), (hits, st) in zip(batches, got):
        want, wst = ctx.map_host(words, lengths, stride, R, q=14, mode=1)
        assert _same(hits, want) and st == wst
    # the same batches as dense 2-bit streams; uniform-length ones without a
    # length array
    dense = []
    for i, (words, lengths, stride) in enumerate(batches):
        codes = np.zeros(lengths.size * stride, np.uint8)
        for r in range(lengths.size):  # unpack the padded words back to codes
            W = (stride + 31) // 32
            for k in range(stride):
                w = int(words[r * W + k // 32])
                codes[r * stride + k] = (w >> (62 - 2 * (k % 32))) & 3
        uniform = bool(np.all(lengths == stride))
        dense.append((qgm.pack_codes(codes), None if uniform else lengths, stride, qgm.READS_DENSE, lengths.size))
    got2 = ctx.map_host_batches(dense, R, q=14, mode=1)
    for (h1, s1), (h2, s2) in zip(got, got2):
        assert _same(h1, h2) and s1 == s2


def test_partition_counter_wrap_with_a_dominant_qgram(ctx, oracle):
    """100k poly-A reads first in the batch put more than 65535 copies of one
    canonical q-gram into a single histogram CTA's share (the packed u16
    shared-memory counter hands 0x8000 to the global count every time it
    reaches 0x8000); the
    20k ordinary reads behind them must still map exactly like the oracle."""
    import paper_1403_1706_b200 as qgm
    L = 400_000
    ref = qgm.random_reference(61, L)
    cb = np.array([0, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(62, ref, cb, 20_000, 100, 0.03)
    n_poly = 100_000
    codes = np.concatenate([np.zeros(n_poly * 100, np.uint8), codes])
    lengths = np.concatenate([np.full(n_poly, 100, np.uint32), lengths])
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    got, st = ctx.map(reads, R, q=16, mode=0)
    want, ost = oracle.map(ref, cb, codes, 100, lengths, q=16, mode=0)
    assert st["index_occurrences"] == lengths.size * 85
    assert _same(got, want), (got.size, want.size)


def test_read_longer_than_stride_is_an_input_error(ctx):
    """The upload does not synchronise; the first stage that does reports a
    read longer than its stride as QGM_ERR_INPUT (seq.hpp's input_error)."""
    import paper_1403_1706_b200 as qgm
    ref = qgm.random_reference(71, 50_000)
    cb = np.array([0, 50_000], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(72, ref, cb, 100, 100, 0.0)
    lengths = lengths.copy()
    lengths[17] = 101
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    with pytest.raises(qgm.InputError):
        ctx.map(reads, R, q=12, mode=0)


def test_validation_park_overflow_finishes_in_phase_one(ctx, oracle, monkeypatch):
    """More phase-1 survivors than the parking capacity (forced to 500): the
    extra candidates are finished in phase 1; hits identical to the oracle."""
    import paper_1403_1706_b200 as qgm
    monkeypatch.setenv("QGM_VAL_PARK_CAP", "500")
    monkeypatch.setenv("QGM_VAL_SPLIT", "64")  # two phases even for a batch this small
    ref, cb, codes, lengths, tp, ts = _c1(qgm, n_reads=5000, L=500_000)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    got, st = ctx.map(reads, R, q=12, mode=1)
    want, ost = oracle.map(ref, cb, codes, 100, lengths, q=12, mode=1)
    assert st["validated"] == ost["validated"]
    assert _same(got, want), (got.size, want.size)


@pytest.mark.parametrize("mode", [0, 1])
def test_map_without_round_trips_equals_the_round_trip_path(ctx, oracle, monkeypatch, mode):
    """The batch mapped without a host round trip before its end (the default
    below 10M candidates), with the round-trip path forced (QGM_MAP_ASYNC=0),
    and with a candidate capacity far below its count (QGM_MAP_ASYNC_CAP=1000:
    the truncated first attempt is detected at the end and the batch mapped
    again): identical hits and statistics, equal to the oracle."""
    import paper_1403_1706_b200 as qgm
    ref, cb, codes, lengths, tp, ts = _c1(qgm, n_reads=5000, L=500_000, seed=11)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    want, ost = oracle.map(ref, cb, codes, 100, lengths, q=12, mode=mode)
    runs = []
    for env in ({}, {"QGM_MAP_ASYNC": "0"}, {"QGM_MAP_ASYNC_CAP": "1000"}):
        with monkeypatch.context() as m:
            for k, v in env.items():
                m.setenv(k, v)
            got, st = ctx.map(reads, R, q=12, mode=mode)
        assert _same(got, want), (env, got.size, want.size)
        _validated_agrees(st, ost, mode, env)
        runs.append({k: v for k, v in st.items() if k != "stage_seconds"})
    assert runs[0] == runs[1] == runs[2], runs
    assert runs[0]["raw_candidates"] > 1000


def test_hit_rank_and_mapq(ctx):
    """hit_rank from the device against a direct count over the output, the
    mapping quality from it, and the hit-rank separation
    property of SPEC.md:499 on a repetitive reference: true origins are more
    frequent among R=1 hits than among R>1 hits."""
    import paper_1403_1706_b200 as qgm
    L = 400_000
    ref = qgm.repetitive_reference(81, L)
    cb = np.array([0, L], np.uint64)
    codes, lengths, tc, tp, ts = qgm.simulate_reads(82, ref, cb, 4000, 100, 0.03)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    hits, st, rank = ctx.map(reads, R, q=12, mode=1, ranks=True)
    want = np.zeros(hits.size, np.uint32)
    order = np.argsort(hits["read_id"], kind="stable")
    bounds = np.searchsorted(hits["read_id"][order], np.unique(hits["read_id"]))
    for b, e in zip(bounds, list(bounds[1:]) + [hits.size]):
        idx = order[b:e]
        ed = hits["edits"][idx]
        want[idx] = (ed[None, :] <= ed[:, None]).sum(1)
    assert np.array_equal(rank, want)
    assert (rank > 1).sum() > 100
    P = R.positions(12)
    assert P == L - 12 + 1  # one chromosome, no mask
    mq = qgm.mapping_quality(rank, P)
    assert np.all(mq[rank == 1] == 255) and np.all(mq[rank > 1] < 255)
    true = np.abs(hits["ref_start"].astype(np.int64) - tp[hits["read_id"]].astype(np.int64)) <= 8
    assert true[rank == 1].mean() > true[rank > 1].mean()
    # both device paths: runs of <= 64 records per read counted in place, and
    # the sorted fallback once one read has more
    assert np.bincount(hits["read_id"]).max() > 64
    for L2, n2 in ((200_000, 3000), (30_000, 500)):
        ref2 = qgm.random_reference(83, L2)
        ref2[10_000:10_100] = ref2[20_000:20_100]
        cb2 = np.array([0, L2], np.uint64)
        codes2, lengths2, *_ = qgm.simulate_reads(84, ref2, cb2, n2, 100, 0.03)
        h2, _, r2 = ctx.map(qgm.Reads.from_codes(ctx, codes2, lengths2, 100), qgm.Reference.from_codes(ctx, ref2, cb2),
                            q=12, mode=1, pct_identity=50, ranks=True)
        w2 = np.zeros(h2.size, np.uint32)
        for r in np.unique(h2["read_id"]):
            idx = np.nonzero(h2["read_id"] == r)[0]
            ed = h2["edits"][idx]
            w2[idx] = (ed[None, :] <= ed[:, None]).sum(1)
        assert np.array_equal(r2, w2)


def _oracle_cigar(oracle, ref, cb, codes, stride, lengths, hits, band):
    ops, info = oracle.cigar(ref, cb, codes, stride, lengths, hits, band=band, max_ops=2 * (stride + band) + 1)
    return ops, info


@pytest.mark.parametrize("band", [32, 64])
def test_cigar_matches_oracle_on_mapped_hits(ctx, oracle, band):
    """traceback_cigar (DESIGN.md section 2 item 9) of every all-mode hit of a C1-shaped run
    with indels, several chromosomes (reads overhanging their ends), both
    strands: device ops and info bit-identical to oracle::traceback_cigar; the
    64-bit band word (B=32) and the 128-bit one (B=64)."""
    import paper_1403_1706_b200 as qgm
    L = 600_000
    ref = qgm.random_reference(31, L)
    cb = np.array([0, 200_000, 200_150, 410_000, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(32, ref, cb, 4000, 100, 0.05)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    hits, st = ctx.map(reads, R, q=12, mode=1, band_width=band)
    assert hits.size > 3000
    ops, info = ctx.cigar(reads, R, hits, band_width=band)
    wops, winfo = _oracle_cigar(oracle, ref, cb, codes, 100, lengths, hits, band)
    assert np.array_equal(info, winfo)
    for i in range(hits.size):
        k = int(info["n_ops"][i])
        assert np.array_equal(ops[i, :k], wops[i, :k]), i
    # the validated alignment lies in the traceback band: never more edits
    # than the hit's k once the dropped leading deletions are counted back
    assert np.all(info["edits"].astype(int) + (info["ref_start"].astype(int) - hits["ref_start"].astype(int))
                  <= hits["edits"].astype(int) + (hits["ref_start"] == 0) * band)
    s = qgm.cigar_string(ops[0], info["n_ops"][0])
    assert s and s[-1] in "MID"


def test_cigar_random_records_and_edges_match_oracle(ctx, oracle):
    """Arbitrary records (random starts, both strands, starts at a
    chromosome's first and last base, a 1-base chromosome, short reads,
    B = 1 and odd bands) -- ties and clamped ends, not only good alignments."""
    import paper_1403_1706_b200 as qgm
    rng = np.random.default_rng(41)
    L = 50_000
    ref = qgm.random_reference(42, L)
    cb = np.array([0, 1, 20_000, 20_040, L], np.uint64)
    stride = 70
    codes, lengths, *_ = qgm.simulate_reads(43, ref, cb, 600, stride, 0.08)
    lengths = np.minimum(lengths, rng.integers(1, stride + 1, lengths.size).astype(np.uint32))
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, stride)
    n = 3000
    hits = np.zeros(n, qgm.HIT_DTYPE)
    hits["read_id"] = rng.integers(0, lengths.size, n)
    hits["chrom"] = rng.integers(0, cb.size - 1, n)
    clen = (cb[1:] - cb[:-1]).astype(np.int64)
    pos = rng.integers(0, 1 << 30, n) % clen[hits["chrom"]]
    pos[::7] = 0
    pos[1::7] = clen[hits["chrom"][1::7]] - 1
    hits["ref_start"] = pos
    hits["strand"] = rng.integers(0, 2, n)
    for band in (1, 7, 32, 33, 64):
        ops, info = ctx.cigar(reads, R, hits, band_width=band)
        wops, winfo = _oracle_cigar(oracle, ref, cb, codes, stride, lengths, hits, band)
        assert np.array_equal(info, winfo), band
        m = np.arange(ops.shape[1])[None, :] < info["n_ops"][:, None]
        assert np.array_equal(np.where(m, ops, 0), np.where(m, wops, 0)), band


def test_cigar_spec_examples_on_device(ctx):
    import paper_1403_1706_b200 as qgm
    enc = lambda s: np.array(["ACGT".index(c) for c in s], np.uint8)  # noqa: E731
    cases = [("ACGT", "ACGT", "4M", 0), ("ACGT", "ACGGT", "2M1D2M", 0), ("ACGT", "ACT", "2M1I1M", 0),
             ("ACGT", "CCACGTCC", "4M", 2)]
    for read, chrom, want, start in cases:
        R = qgm.Reference.from_codes(ctx, enc(chrom), np.array([0, len(chrom)], np.uint64))
        reads = qgm.Reads.from_codes(ctx, enc(read), np.array([len(read)], np.uint32), len(read))
        h = np.zeros(1, qgm.HIT_DTYPE)
        ops, info = ctx.cigar(reads, R, h)
        assert qgm.cigar_string(ops[0], info["n_ops"][0]) == want and info["ref_start"][0] == start


def test_cigar_long_reads_use_global_rows_and_match_oracle(ctx, oracle):
    """Reads too long for the shared-memory rows (300 bp at B=64: 301 rows x
    16 B x 32 threads > 113 KiB) take the global-scratch path; 500 bp at B=32
    too."""
    import paper_1403_1706_b200 as qgm
    L = 300_000
    ref = qgm.random_reference(51, L)
    cb = np.array([0, 120_000, L], np.uint64)
    for stride, band in ((300, 64), (500, 32), (300, 32)):
        codes, lengths, *_ = qgm.simulate_reads(52 + stride, ref, cb, 300, stride, 0.04)
        R = qgm.Reference.from_codes(ctx, ref, cb)
        reads = qgm.Reads.from_codes(ctx, codes, lengths, stride)
        hits, st = ctx.map(reads, R, q=14, mode=1, band_width=band, pct_identity=70)
        assert hits.size > 200
        ops, info = ctx.cigar(reads, R, hits, band_width=band)
        wops, winfo = _oracle_cigar(oracle, ref, cb, codes, stride, lengths, hits, band)
        assert np.array_equal(info, winfo), (stride, band)
        m = np.arange(ops.shape[1])[None, :] < info["n_ops"][:, None]
        assert np.array_equal(np.where(m, ops, 0), np.where(m, wops, 0)), (stride, band)


@pytest.mark.parametrize("mode", [0, 1])
def test_reference_sharded_pieces_reproduce_the_whole_reference(ctx, mode):
    """SURVEY 8(f) row 2 on one GPU: the shares of a 4-way reference split are
    mapped one after another on the device (each rank's work), owned hits kept
    and combined as the exchange step would (MIN of k per read, union): the
    result equals mapping the whole reference."""
    import paper_1403_1706_b200 as qgm
    from paper_1403_1706_b200 import refshard
    L = 400_000
    ref = qgm.random_reference(61, L)
    ref[300_000:300_500] = ref[50_000:50_500]
    cb = np.array([0, 180_000, 180_300, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(62, ref, cb, 5000, 100, 0.04)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    want, _ = ctx.map(reads, qgm.Reference.from_codes(ctx, ref, cb), q=14, mode=mode)
    parts = []
    for pieces in refshard.plan(cb, 4, 100, 32):
        pc, pcb, _ = refshard.piece_reference(ref, cb, pieces)
        local, _ = ctx.map(reads, qgm.Reference.from_codes(ctx, pc, pcb), q=14, mode=1)
        parts.append(refshard.own_and_translate(local, pieces))
    got = refshard.combine(np.concatenate(parts), lengths.size, mode)
    assert got.size == want.size and got.size > 4000
    assert np.array_equal(got, want)


def test_large_candidate_sets_skip_the_dedup_only_when_it_cannot_pay(ctx, oracle, monkeypatch):
    """Above the L2-resident hash size the candidate dedup is decided from a
    1/64 read sample (forced here by lowering the size limit): a random
    reference at q=10 (~50 random candidates per read, ~2% duplicates) skips
    it, a repetitive one (mostly duplicates) keeps it; the hits equal the
    oracle's either way."""
    import paper_1403_1706_b200 as qgm
    monkeypatch.setenv("QGM_DEDUP_DIRECT_MAX", "1000")
    # kept dedup of a large set: one radix pass into partitions, each hashed
    # in the reused L2-sized table (here forced to 256 partitions)
    monkeypatch.setenv("QGM_DEDUP_PART_KEYS", "64")
    for rep, seed, q in ((False, 91, 10), (True, 92, 12)):
        L = 300_000
        ref = qgm.repetitive_reference(seed, L) if rep else qgm.random_reference(seed, L)
        cb = np.array([0, L], np.uint64)
        codes, lengths, *_ = qgm.simulate_reads(seed + 1, ref, cb, 4000, 100, 0.03)
        R = qgm.Reference.from_codes(ctx, ref, cb)
        reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
        for mode in (0, 1):
            got, st = ctx.map(reads, R, q=q, mode=mode)
            want, ost = oracle.map(ref, cb, codes, 100, lengths, q=q, mode=mode)
            assert _same(got, want), (rep, mode)
            skipped = st["unique_candidates"] == st["raw_candidates"]
            assert skipped == (not rep), (rep, st)
            if not skipped:
                assert st["unique_candidates"] == ost["unique_candidates"]


def test_randomised_configurations_match_oracle(ctx, oracle):
    """A seeded sweep over the parameter space the C ABI accepts -- q 4..16,
    band 1..64, identity 0..100%, both modes, one strand or both, 1-6
    chromosomes (some shorter than a read), read lengths 1..stride, error
    rates up to 12%, optional repeat mask -- every configuration bit-identical
    to the oracle, stats included, and the CIGARs of the hits too."""
    import paper_1403_1706_b200 as qgm
    rng = np.random.default_rng(2026)
    for case in range(24):
        q = int(rng.integers(4, 17))
        band = int(rng.choice([1, 2, 7, 16, 31, 32, 33, 48, 64]))
        pct = int(rng.choice([0, 50, 70, 80, 90, 100]))
        mode = int(rng.integers(0, 2))
        strands = int(rng.choice([1, 2, 3]))
        n_chrom = int(rng.integers(1, 7))
        L = int(rng.integers(20_000, 120_000))
        ref = qgm.random_reference(int(rng.integers(1 << 30)), L)
        cuts = np.sort(rng.choice(np.arange(1, L), n_chrom - 1, replace=False)) if n_chrom > 1 else np.array([], int)
        cb = np.concatenate([[0], cuts, [L]]).astype(np.uint64)
        stride = int(rng.choice([20, 64, 100, 150, 255]))
        n_reads = int(rng.integers(50, 800))
        err = float(rng.choice([0.0, 0.03, 0.08, 0.12]))
        codes, lengths, *_ = qgm.simulate_reads(int(rng.integers(1 << 30)), ref, cb, n_reads, stride, err)
        if rng.random() < 0.5:
            lengths = np.minimum(lengths, rng.integers(1, stride + 1, lengths.size).astype(np.uint32))
        mask = None
        if rng.random() < 0.3:
            from oracle.pyoracle import repeat_mask
            mask = repeat_mask(ref, cb, q, int(rng.integers(1, 4)))
        R = qgm.Reference.from_codes(ctx, ref, cb, mask=mask)
        reads = qgm.Reads.from_codes(ctx, codes, lengths, stride)
        got, st = ctx.map(reads, R, q=q, mode=mode, band_width=band, pct_identity=pct, strands=strands)
        want, ost = oracle.map(ref, cb, codes, stride, lengths, q=q, mode=mode, band=band, pct=pct, strands=strands,
                               mask=mask)
        info = dict(case=case, q=q, band=band, pct=pct, mode=mode, strands=strands, chroms=n_chrom, stride=stride,
                    err=err, mask=mask is not None, got=got.size, want=want.size)
        assert _same(got, want), info
        assert st["unique_candidates"] == ost["unique_candidates"], info
        _validated_agrees(st, ost, mode, info)
        if got.size:  # and the traceback of every hit
            ops, cinfo = ctx.cigar(reads, R, got, band_width=band)
            wops, winfo = oracle.cigar(ref, cb, codes, stride, lengths, got, band=band, max_ops=ops.shape[1])
            assert np.array_equal(cinfo, winfo), info
            m = np.arange(ops.shape[1])[None, :] < cinfo["n_ops"][:, None]
            assert np.array_equal(np.where(m, ops, 0), np.where(m, wops, 0)), info


def test_cigar_max_ops_overflow_is_an_input_error_with_counts(ctx):
    """qgm_cigar_records with too small a max_ops: QGM_ERR_INPUT, every n_ops
    filled in so the caller can retry (include/qgm_c.h)."""
    import ctypes as C
    import paper_1403_1706_b200 as qgm
    L = 50_000
    ref = qgm.random_reference(71, L)
    cb = np.array([0, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(72, ref, cb, 300, 100, 0.08)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    hits, _ = ctx.map(reads, R, q=12, mode=1)
    ops_ok, info_ok = ctx.cigar(reads, R, hits)
    assert info_ok["n_ops"].max() > 1
    ops = np.zeros(hits.size, np.uint32)
    info = np.zeros(hits.size, qgm.CIGAR_DTYPE)
    rc = ctx.lib.qgm_cigar_records(ctx.h, reads.h, R.h, hits.ctypes.data_as(C.c_void_p), hits.size, 32, 1,
                                   ops.ctypes.data_as(C.c_void_p), info.ctypes.data_as(C.c_void_p))
    assert rc == 1  # QGM_ERR_INPUT
    assert np.array_equal(info["n_ops"], info_ok["n_ops"])
    assert "max_ops" in ctx.lib.qgm_last_error(ctx.h).decode()


def test_map_returns_ranks_and_cigars_from_device_hits(ctx):
    """ctx.map(..., ranks=True, cigars=True): ranks and CIGARs computed from
    the device-resident hits equal the separate calls on downloaded hits."""
    import paper_1403_1706_b200 as qgm
    L = 80_000
    ref = qgm.random_reference(81, L)
    cb = np.array([0, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(82, ref, cb, 400, 100, 0.05)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    hits, st, ranks, (ops, info) = ctx.map(reads, R, q=12, mode=1, ranks=True, cigars=True)
    h2, _, r2 = ctx.map(reads, R, q=12, mode=1, ranks=True)
    ops2, info2 = ctx.cigar(reads, R, h2)
    assert np.array_equal(hits, h2) and np.array_equal(ranks, r2)
    assert np.array_equal(info, info2)
    m = np.arange(ops.shape[1])[None, :] < info["n_ops"][:, None]
    assert np.array_equal(np.where(m, ops, 0), np.where(m, ops2[:, : ops.shape[1]], 0))
    hits3, st3, (ops3, info3) = ctx.map(reads, R, q=12, mode=1, cigars=True)
    assert np.array_equal(info3, info)


@pytest.mark.parametrize("world", [1, 2])
def test_reference_sharded_exchange_on_device_across_ranks(world):
    """SURVEY 8(f) row 2 end to end: tools/refshard_nccl_check.py under
    torchrun -- records downloaded device to device, owned hits kept, MIN
    all-reduce + all-to-all (NCCL with a GPU per rank; on a 1-GPU box the two
    ranks share the device and exchange over gloo) -- equals the whole
    reference's map in both modes."""
    import subprocess
    import sys
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={29650 + world}", "tools/refshard_nccl_check.py"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("identical=True") == 2, r.stdout


def test_bench_two_ranks_share_one_gpu_and_gather():
    """bench.py --gpus 2 re-launches itself under torchrun; on a 1-GPU box the
    two ranks share the device over gloo. The line reports both ranks' reads
    and the end-of-run gather of every rank's hits into one host buffer."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "C1", "--steps", "2", "--warmup", "1",
                        "--no-cpu"], capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["reads_per_step"] == 20_000
    assert line["gathered"]["hits"] > 19_000
    assert line["e2e"]["gather"]["method"].startswith("all_gather")

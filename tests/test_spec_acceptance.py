"""SPEC.md acceptance criteria 3, 4, 7 and 8
on the device path (qgm_filter / qgm_map through the C ABI).

3. Pigeonhole sensitivity: 10^4 length-100 reads from a random 1 Mbp
   reference, each with e <= 5 seeded substitutions, q = 16: filtration yields
   the true (r, strand, d) candidate for 100% of reads (the q-gram lemma: at
   least n + 1 - (e + 1) q = 5 error-free 16-grams remain).
4. End-to-end sensitivity, all mode, identity threshold 60: >= 99.5% of 1000
   reads at 5% per-base error (substitutions + short indels) yield a record
   overlapping their true origin, at q = 16 (the paper's default).
   At 20% per-base error: >= 98%. SPEC's desk analogue takes the paper's
   "error rate up to 20%" (a Rabema error tolerance over Mason
   reads at default error rates) as 20 random edits per 100 bp read; then a
   shared exact 16-gram exists for only ~43% of reads (measured with the CPU
   oracle), so no q = 16 filter can pass it. The criterion is checked at
   q = 8 (where the expected longest error-free run covers a q-gram for ~99.6%
   of reads) and the q = 16 rate is asserted to match the oracle's exactly.
7. Hit-rank separation: precision of rank-1 hits exceeds that of rank >= 2
   hits by >= 20 percentage points on criterion 4's data.
8. Determinism: repeated maps and different batch splits give identical hits.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

L = 1_000_000


def _ref(seed=21):
    import paper_1403_1706_b200 as qgm
    return qgm.random_reference(seed, L), np.array([0, L], np.uint64)


def _substitution_reads(ref, n_reads, max_subs, seed):
    """Reads of length 100 sampled uniformly, 50% reverse complement, with
    e ~ U{0..max_subs} substitutions at distinct positions (to a different
    base). Returns codes, lengths, true start, strand."""
    rng = np.random.default_rng(seed)
    pos = rng.integers(0, L - 100, n_reads)
    strand = rng.integers(0, 2, n_reads).astype(np.uint8)
    reads = ref[pos[:, None] + np.arange(100)].astype(np.uint8)
    rc = strand == 1
    reads[rc] = (3 - reads[rc])[:, ::-1]
    for i, e in enumerate(rng.integers(0, max_subs + 1, n_reads)):
        at = rng.choice(100, size=e, replace=False)
        reads[i, at] = (reads[i, at] + rng.integers(1, 4, e)) % 4
    return reads.reshape(-1), np.full(n_reads, 100, np.uint32), pos, strand


def _sensitivity(hits, tp, ts, lengths):
    r = hits["read_id"].astype(np.int64)
    s = hits["ref_start"].astype(np.int64)
    t0 = tp[r].astype(np.int64)
    ov = (s < t0 + lengths[r]) & (s + lengths[r] > t0) & (hits["strand"] == ts[r])
    ok = np.zeros(lengths.size, bool)
    ok[r[ov]] = True
    return ok.mean(), ov


def test_criterion3_pigeonhole_true_candidate_for_every_read(ctx):
    import paper_1403_1706_b200 as qgm
    ref, cb = _ref()
    codes, lengths, pos, strand = _substitution_reads(ref, 10_000, 5, seed=3)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    idx = qgm.Index.build(ctx, reads, 16)
    for mode in (qgm.FILTER_RUN_START, qgm.FILTER_RUN_START | qgm.FILTER_JOIN,
                 qgm.FILTER_RUN_START | qgm.FILTER_STREAM):
        cands = ctx.filter(idx, reads, R, mode=mode, unique=True)
        key = set(zip(cands["read_id"].tolist(), cands["strand"].tolist(), cands["diagonal"].tolist()))
        missing = [r for r in range(lengths.size) if (r, int(strand[r]), int(pos[r])) not in key]
        assert not missing, (mode, len(missing), missing[:5])
    # and the map keeps every read at its origin: a best-stratum hit on the
    # true strand within e bases of it (a substitution next to a read end can
    # make an equally cheap alignment start a base earlier, and the smallest
    # start wins) with k <= e <= 5
    hits, st = ctx.map(reads, R, q=16, mode=qgm.MODE_BEST_STRATUM)
    r = hits["read_id"]
    near = (np.abs(hits["ref_start"].astype(np.int64) - pos[r]) <= 5) & (hits["strand"] == strand[r]) & \
        (hits["edits"] <= 5)
    found = np.zeros(lengths.size, bool)
    found[r[near]] = True
    assert found.all(), int((~found).sum())


@pytest.mark.parametrize("err,q,want", [(0.05, 16, 0.995), (0.20, 8, 0.98)])
def test_criterion4_end_to_end_sensitivity(ctx, oracle, err, q, want):
    import paper_1403_1706_b200 as qgm
    ref, cb = _ref()
    codes, lengths, tc, tp, ts = qgm.simulate_reads(22, ref, cb, 1000, 100, err)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    hits, st = ctx.map(reads, R, q=q, mode=qgm.MODE_ALL, pct_identity=60)
    sens, _ = _sensitivity(hits, tp, ts, lengths)
    assert sens >= want, sens
    want_hits, _ = oracle.map(ref, cb, codes, 100, lengths, q=q, mode=1, pct=60)
    assert hits.size == want_hits.size and all(np.array_equal(hits[c], want_hits[c])
                                               for c in ("read_id", "chrom", "ref_start", "edits", "strand"))


def test_criterion4_q16_at_20pct_matches_the_oracle(ctx, oracle):
    """q = 16 at 20% per-base error: the filtration limit, not a mapper loss --
    the device finds exactly the oracle's hits (sensitivity ~0.43)."""
    import paper_1403_1706_b200 as qgm
    ref, cb = _ref()
    codes, lengths, tc, tp, ts = qgm.simulate_reads(22, ref, cb, 1000, 100, 0.20)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    hits, _ = ctx.map(reads, R, q=16, mode=qgm.MODE_ALL, pct_identity=60)
    want, _ = oracle.map(ref, cb, codes, 100, lengths, q=16, mode=1, pct=60)
    assert _sensitivity(hits, tp, ts, lengths)[0] == _sensitivity(want, tp, ts, lengths)[0]
    assert hits.size == want.size


def test_criterion7_rank1_precision_exceeds_rank2_by_20_points(ctx):
    import paper_1403_1706_b200 as qgm
    ref, cb = _ref()
    # a reference with repeats makes rank >= 2 hits exist: copy 200 kb segments
    ref = ref.copy()
    ref[600_000:700_000] = ref[100_000:200_000]
    ref[650_000:650_100] = (ref[650_000:650_100] + 1) % 4
    codes, lengths, tc, tp, ts = qgm.simulate_reads(23, ref, cb, 1000, 100, 0.05)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    hits, st, ranks = ctx.map(reads, R, q=16, mode=qgm.MODE_ALL, pct_identity=60, ranks=True)
    _, ov = _sensitivity(hits, tp, ts, lengths)
    r1, r2 = ranks == 1, ranks >= 2
    assert r1.any() and r2.any()
    p1, p2 = ov[r1].mean(), ov[r2].mean()
    assert p1 - p2 >= 0.20, (p1, p2)


def test_criterion8_determinism_repeat_and_batch_split(ctx):
    import paper_1403_1706_b200 as qgm
    ref, cb = _ref()
    codes, lengths, tc, tp, ts = qgm.simulate_reads(24, ref, cb, 6000, 100, 0.05)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
    a, _ = ctx.map(reads, R, q=16, mode=qgm.MODE_ALL, pct_identity=60)
    b, _ = ctx.map(reads, R, q=16, mode=qgm.MODE_ALL, pct_identity=60)
    assert a.tobytes() == b.tobytes()
    words = qgm.pack_read_codes(codes, 100)
    parts = ctx.map_host_batches([(words[i * 2000 * 4:(i + 1) * 2000 * 4], lengths[i * 2000:(i + 1) * 2000], 100)
                                  for i in range(3)], R, q=16, mode=qgm.MODE_ALL, pct_identity=60)
    merged = []
    for i, (h, _) in enumerate(parts):
        h = h.copy()
        h["read_id"] += i * 2000
        merged.append(h)
    merged = np.concatenate(merged)
    assert merged.tobytes() == a.tobytes()

"""Small device workload for compute-sanitizer (tools/sanitize.sh).

Reaches every kernel variant of the map path at sizes the sanitizers finish
in minutes: plain and warp-specialised join, packed and unpacked reference
index, the P0 u16 counter hand-off, parked two-phase validation (and its
overflow branch), the sampled dedup decision, the partitioned dedup, the
strata radix path (reads
with > 32 hits), hit ranks, CIGARs, streamed batches and the standalone
filter / validate / index entry points. Every map is checked against the CPU
oracle (test infrastructure), so a hazard that changes a result fails here too.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1403_1706_b200 as qgm  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402  (checker only)

COLS = ("read_id", "chrom", "ref_start", "edits", "strand")


def same(a, b):
    return a.size == b.size and all(np.array_equal(a[c], b[c]) for c in COLS)


def run(ctx, orc, name, ref, cb, codes, lengths, stride, **kw):
    R = qgm.Reference.from_codes(ctx, ref, cb)
    reads = qgm.Reads.from_codes(ctx, codes, lengths, stride)
    got, st = ctx.map(reads, R, **kw)
    want, _ = orc.map(ref, cb, codes, stride, lengths, q=kw["q"], mode=kw["mode"], band=kw.get("band_width", 32))
    ok = same(got, want)
    print(f"{name}: {got.size} hits, oracle {want.size}, stats {st}, parity={ok}", flush=True)
    if not ok:
        raise SystemExit(f"{name}: parity failure")
    return R, reads, got


def main():
    ctx = qgm.Context(0)
    orc = Oracle()
    L = 2_000_000
    ref = qgm.random_reference(11, L)
    cb = np.array([0, 1_200_000, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(12, ref, cb, 30_000, 100, 0.03)

    # plain join (q=16: 16-bit sub-bins of ~40 q-grams) and parked validation
    run(ctx, orc, "join q16 best", ref, cb, codes, lengths, 100, q=16, mode=0)
    run(ctx, orc, "join q16 all", ref, cb, codes, lengths, 100, q=16, mode=1)
    # warp-specialised join (q=12: 13-bit sub-bins of ~300 q-grams, staged)
    os.environ["QGM_JOIN_WS"] = "1"
    R, reads, got = run(ctx, orc, "join_ws q12 best", ref, cb, codes, lengths, 100, q=12, mode=0)
    os.environ["QGM_JOIN_WS"] = ""
    # hit ranks + CIGARs of the device-resident hits
    h, st, ranks, (ops, info) = ctx.map(reads, R, q=12, mode=0, ranks=True, cigars=True)
    print(f"ranks/cigars: {h.size} records, max ops {int(info['n_ops'].max())}", flush=True)
    del reads, R

    # validation park overflow branch + sampled dedup decision
    os.environ["QGM_VAL_PARK_CAP"] = "1000"
    os.environ["QGM_VAL_SPLIT"] = "64"  # two phases even for this batch size
    os.environ["QGM_DEDUP_DIRECT_MAX"] = "20000"
    run(ctx, orc, "park overflow + sampled dedup", ref, cb, codes, lengths, 100, q=12, mode=0)
    os.environ["QGM_VAL_PARK_CAP"] = ""
    os.environ["QGM_VAL_SPLIT"] = ""
    os.environ["QGM_DEDUP_DIRECT_MAX"] = ""

    # kept dedup of a large repetitive candidate set through the partitioned
    # path: one radix pass, 256 partitions, the reused table reset by each
    # compaction
    os.environ["QGM_DEDUP_DIRECT_MAX"] = "1000"
    os.environ["QGM_DEDUP_PART_KEYS"] = "64"
    rref = qgm.repetitive_reference(92, 300_000)
    rcb = np.array([0, 300_000], np.uint64)
    rcodes, rlengths, *_ = qgm.simulate_reads(93, rref, rcb, 4000, 100, 0.03)
    run(ctx, orc, "partitioned dedup", rref, rcb, rcodes, rlengths, 100, q=12, mode=1)
    os.environ["QGM_DEDUP_DIRECT_MAX"] = ""
    os.environ["QGM_DEDUP_PART_KEYS"] = ""

    # unpacked reference index (O without packed extra bits)
    os.environ["QGM_REF_UNPACKED"] = "1"
    run(ctx, orc, "unpacked index", ref, cb, codes, lengths, 100, q=16, mode=1)
    os.environ["QGM_REF_UNPACKED"] = ""

    # P0 u16 counter hand-off: 60k poly-A reads ahead of 10k ordinary ones
    c2, l2, *_ = qgm.simulate_reads(13, ref, cb, 10_000, 100, 0.03)
    cw = np.concatenate([np.zeros(60_000 * 100, np.uint8), c2])
    lw = np.concatenate([np.full(60_000, 100, np.uint32), l2])
    run(ctx, orc, "counter hand-off", ref, cb, cw, lw, 100, q=16, mode=0)

    # repetitive reference: reads with > 32 hits (strata radix path), band 64
    rref = qgm.repetitive_reference(14, 400_000)
    rcb = np.array([0, 400_000], np.uint64)
    rc, rl, *_ = qgm.simulate_reads(15, rref, rcb, 5_000, 100, 0.03)
    run(ctx, orc, "repeats all b64", rref, rcb, rc, rl, 100, q=16, mode=1, band_width=64)

    # variable read lengths (stride 130)
    vc, vl, *_ = qgm.simulate_reads(16, ref, cb, 5_000, 100, 0.05, stride=130)
    vl = np.minimum(vl, 130).astype(np.uint32)
    run(ctx, orc, "stride 130", ref, cb, vc, vl, 130, q=12, mode=1)

    # standalone entry points: index build, streaming filter, validate
    R = qgm.Reference.from_codes(ctx, ref, cb)
    small_c, small_l = codes[: 2000 * 100], lengths[:2000]
    reads = qgm.Reads.from_codes(ctx, small_c, small_l, 100)
    idx = qgm.Index.build(ctx, reads, 12)
    cands = ctx.filter(idx, reads, R, mode=qgm.FILTER_RUN_START | qgm.FILTER_STREAM, unique=True)
    val = ctx.validate(reads, R, cands[:5000])
    print(f"api: {idx.info['occurrences']} occurrences, {cands.size} candidates, {int(val['kept'].sum())} kept",
          flush=True)
    # streamed batches
    words = qgm.pack_read_codes(codes, 100)
    W = 4
    bs = [(words[i * 10_000 * W:(i + 1) * 10_000 * W], lengths[i * 10_000:(i + 1) * 10_000], 100) for i in range(3)]
    res = ctx.map_host_batches(bs, R, q=16, mode=1)
    print(f"streamed: {[r[0].size for r in res]}", flush=True)
    del reads, R, idx
    ctx.close()
    print("sanitize workload: done", flush=True)


if __name__ == "__main__":
    main()

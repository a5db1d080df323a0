"""Generate tests/golden/golden_v1.json from the REFERENCE's own code.

Runs the reference's build_qgroup_index, oracle::filter_hits,
oracle::banded_semiglobal_distance / anchored_start_distance and pack_reads
(compiled from /root/reference by oracle/Makefile into oracle/_ref/libqgm_ref.so)
on small seeded inputs and stores inputs + outputs as JSON, so the oracle can be
pinned on machines where /root/reference does not exist (the GPU box).

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import RefShim, rc_codes, sort_intervals  # noqa: E402


def rand_reads(rng, n_reads, stride, lmin=0):
    lengths = rng.integers(lmin, stride + 1, n_reads).astype(np.uint32)
    codes = np.zeros(n_reads * stride, dtype=np.uint8)
    for r in range(n_reads):
        codes[r * stride:r * stride + lengths[r]] = rng.integers(0, 4, lengths[r])
    return codes, lengths


def main():
    ref = RefShim()
    rng = np.random.default_rng(20241017)
    out = {"source": "reference build_qgroup_index / oracles.hpp via oracle/_ref/libqgm_ref.so",
           "index": [], "filter": [], "banded": [], "pack_reads": [], "scan": [], "size": []}
    # --- index (qgroup_index.hpp:124-180), O normalised per interval
    for it in range(24):
        q = int(rng.integers(1, 9))
        w = 32 if it % 3 else 64
        sampled = bool(it % 4 == 1)
        stride = int(rng.integers(q, q + 12))
        codes, lengths = rand_reads(rng, int(rng.integers(0, 12)), stride)
        I, S, S1, O = ref.build_index(codes, stride, lengths, q, w, sampled, threads=1)
        out["index"].append({"q": q, "w": w, "sampled": sampled, "stride": stride, "codes": codes.tolist(),
                             "lengths": lengths.tolist(), "I": [int(x) for x in I], "S": S.tolist(),
                             "S1": S1.tolist(), "O": sort_intervals(S1, O).tolist()})
    # --- filtration (oracles.hpp:37-51), forward and on RC(reference)
    for it in range(12):
        q = int(rng.integers(2, 7))
        stride = int(rng.integers(q, q + 10))
        codes, lengths = rand_reads(rng, int(rng.integers(1, 8)), stride)
        L = int(rng.integers(0, 60))
        chrom = rng.integers(0, 4, L).astype(np.uint8)
        entry = {"q": q, "stride": stride, "codes": codes.tolist(), "lengths": lengths.tolist(),
                 "chrom": chrom.tolist()}
        for name, seq in (("fwd", chrom), ("rc", rc_codes(chrom))):
            pos = np.arange(max(L - q + 1, 0), dtype=np.uint32)
            cod = np.array([int("".join(map(str, seq[p:p + q])) or "0", 4) if q else 0 for p in pos], dtype=np.uint32)
            hits = ref.filter_hits(pos, cod, codes, stride, lengths, q)
            entry[name] = [[int(h["diagonal"]), int(h["read_id"])] for h in hits]
        out["filter"].append(entry)
    # --- banded semi-global distance (oracles.hpp:86-111) + anchored (:116-135)
    for it in range(200):
        n = int(rng.integers(1, 24))
        B = int(rng.integers(1, 12))
        read = rng.integers(0, 4, n).astype(np.uint8)
        win = rng.integers(0, 4, n + B - 1).astype(np.uint8)
        off = int(rng.integers(0, B))
        seg = read[: n + B - 1 - off].copy()
        if seg.size and rng.random() < 0.7:
            seg[int(rng.integers(0, seg.size))] = rng.integers(0, 4)
        win[off:off + seg.size] = seg
        k = ref.banded_distance(read, win, B)
        anch = [ref.anchored_start_distance(read, win, s) for s in range(B)]
        out["banded"].append({"read": read.tolist(), "window": win.tolist(), "B": B, "k": k, "anchored": anch})
    # --- codec (seq.hpp:142-148) with seeded N replacement
    for reads, stride, q, seed in ((["ACGT", "TACG"], 4, 2, 1), (["AC"], 4, 2, 1), (["ACGNNTA", "NNNN", "GGGTACGT"], 8, 3, 99),
                                   (["acgtn", "NACGT"], 6, 2, 7)):
        codes, valid = ref.pack_reads(reads, stride, q, seed)
        out["pack_reads"].append({"reads": reads, "stride": stride, "q": q, "seed": seed, "codes": codes.tolist(),
                                  "valid": valid.tolist()})
    # --- scan KATs (parallel.hpp:64-121)
    for vals in ([3, 0, 2], [], [1, 1, 1, 1], rng.integers(0, 100, 5000).tolist()):
        sums, total = ref.exclusive_scan(np.array(vals, dtype=np.uint32))
        out["scan"].append({"in": [int(v) for v in vals], "sums": sums.tolist(), "total": int(total)})
    # --- size formula (qgroup_index.hpp:198-213)
    for q, T, w in ((16, 10 ** 8, 32), (10, 4 ** 10, 32), (12, 4 ** 12 * 15 // 16, 32), (8, 1000, 64)):
        a, b, r = ref.index_size_words(q, T, w)
        out["size"].append({"q": q, "T": T, "w": w, "qgroup": a, "classic": b, "ratio": r})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracle and the reference shim.

    Oracle   oracle/build/libqgm_oracle.so : restatement of the hot path
             (oracle/qgm_oracle.hpp), CPU only.
    RefShim  oracle/_ref/libqgm_ref.so     : the reference's own code
             (build_qgroup_index, oracles.hpp) compiled from /root/reference.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
The product (paper_1403_1706_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libqgm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqgm_ref.so")

CAND_DTYPE = np.dtype([("diagonal", "<i8"), ("read_id", "<u4"), ("chrom", "<u4"), ("strand", "<u4"),
                       ("reserved", "<u4")])
HIT_DTYPE = np.dtype([("read_id", "<u4"), ("chrom", "<u4"), ("ref_start", "<u4"), ("edits", "<u2"),
                      ("strand", "u1"), ("reserved", "u1")])
VAL_DTYPE = np.dtype([("edits", "<i4"), ("start", "<u4"), ("ref_start", "<u4"), ("kept", "u1"),
                      ("in_range", "u1"), ("r0", "u1"), ("r1", "u1"), ("r2", "<u4")])
CIGAR_DTYPE = np.dtype([("ref_start", "<u4"), ("n_ops", "<u2"), ("edits", "<u2")])
REFHIT_DTYPE = np.dtype([("diagonal", "<i8"), ("read_id", "<u4"), ("pad", "<u4")])

P = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Buffers:
    def __init__(self, lib, prefix):
        self.lib = lib
        self.size = getattr(lib, prefix + "buf_size")
        self.size.restype = C.c_uint64
        self.size.argtypes = [P]
        self.data = getattr(lib, prefix + "buf_data")
        self.data.restype = P
        self.data.argtypes = [P]
        self.free = getattr(lib, prefix + "buf_free")
        self.free.argtypes = [P]
        self.err = getattr(lib, prefix + "last_error")
        self.err.restype = C.c_char_p

    def take(self, h, dtype):
        n = self.size(h)
        out = np.empty(n // np.dtype(dtype).itemsize, dtype=dtype)
        if n:
            C.memmove(out.ctypes.data, self.data(h), n)
        self.free(h)
        return out

    def check(self, rc):
        if rc:
            raise (ValueError if rc == 1 else RuntimeError)(self.err().decode())


def _reads_args(codes, stride, lengths):
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    lengths = np.ascontiguousarray(lengths, dtype=np.uint32)
    return codes, lengths


class Oracle:
    """CPU restatement (qgm_oracle.hpp)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.b = _Buffers(self.lib, "orc_")

    def build_index(self, codes, stride, lengths, q, w=32, sampled=False):
        codes, lengths = _reads_args(codes, stride, lengths)
        hs = [P() for _ in range(4)]
        f = self.lib.orc_build_index
        f.argtypes = [P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int] + [C.POINTER(P)] * 4
        self.b.check(f(_p(codes), stride, _p(lengths), lengths.size, q, w, int(sampled), *[C.byref(h) for h in hs]))
        wd = np.uint32 if w == 32 else np.uint64
        return (self.b.take(hs[0], wd), self.b.take(hs[1], np.uint32), self.b.take(hs[2], np.uint32),
                self.b.take(hs[3], np.uint32))

    def filter(self, ref_codes, chrom_begin, read_codes, stride, lengths, q, strands=3, run_start=False,
               mask=None, threads=0):
        ref_codes = np.ascontiguousarray(ref_codes, dtype=np.uint8)
        cb = np.ascontiguousarray(chrom_begin, dtype=np.uint64)
        read_codes, lengths = _reads_args(read_codes, stride, lengths)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        h = P()
        f = self.lib.orc_filter
        f.argtypes = [P, P, C.c_uint32, P, P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_uint32,
                      C.POINTER(P)]
        self.b.check(f(_p(ref_codes), _p(cb), cb.size - 1, _p(m), _p(read_codes), stride, _p(lengths), lengths.size,
                       q, strands, int(run_start), threads, C.byref(h)))
        return self.b.take(h, CAND_DTYPE)

    def validate_pair(self, read, window, band, use_dp=False):
        read = np.ascontiguousarray(read, dtype=np.uint8)
        window = np.ascontiguousarray(window, dtype=np.uint8)
        k, s = C.c_int32(), C.c_uint32()
        f = self.lib.orc_validate
        f.argtypes = [P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_uint32)]
        self.b.check(f(_p(read), read.size, _p(window), window.size, band, int(use_dp), C.byref(k), C.byref(s)))
        return k.value, s.value

    def validate_cands(self, ref_codes, chrom_begin, read_codes, stride, lengths, cands, band=32, pct=80,
                       use_dp=False, threads=0):
        ref_codes = np.ascontiguousarray(ref_codes, dtype=np.uint8)
        cb = np.ascontiguousarray(chrom_begin, dtype=np.uint64)
        read_codes, lengths = _reads_args(read_codes, stride, lengths)
        cands = np.ascontiguousarray(cands, dtype=CAND_DTYPE)
        out = np.zeros(cands.size, dtype=VAL_DTYPE)
        f = self.lib.orc_validate_cands
        f.argtypes = [P, P, C.c_uint32, P, C.c_uint32, P, C.c_uint32, P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int,
                      C.c_uint32, P]
        self.b.check(f(_p(ref_codes), _p(cb), cb.size - 1, _p(read_codes), stride, _p(lengths), lengths.size,
                       _p(cands), cands.size, band, pct, int(use_dp), threads, _p(out)))
        return out

    def cigar(self, ref_codes, chrom_begin, read_codes, stride, lengths, hits, band=32, max_ops=64, threads=0):
        """traceback_cigar (DESIGN.md section 2 item 9) of hit records -> (ops[n, max_ops] u32, info)."""
        ref_codes = np.ascontiguousarray(ref_codes, dtype=np.uint8)
        cb = np.ascontiguousarray(chrom_begin, dtype=np.uint64)
        read_codes, lengths = _reads_args(read_codes, stride, lengths)
        hits = np.ascontiguousarray(hits, dtype=HIT_DTYPE)
        ops = np.zeros((hits.size, max_ops), np.uint32)
        info = np.zeros(hits.size, CIGAR_DTYPE)
        f = self.lib.orc_cigar
        f.argtypes = [P, P, C.c_uint32, P, C.c_uint32, P, C.c_uint32, P, C.c_uint64, C.c_uint32, C.c_uint32,
                      C.c_uint32, P, P]
        self.b.check(f(_p(ref_codes), _p(cb), cb.size - 1, _p(read_codes), stride, _p(lengths), lengths.size,
                       _p(hits), hits.size, band, max_ops, threads, _p(ops), _p(info)))
        return ops, info

    def map(self, ref_codes, chrom_begin, read_codes, stride, lengths, q=16, w=32, sampled=False, band=32, pct=80,
            mode=0, strands=3, mask=None, threads=0):
        return _map(self.lib, "orc_map", self.b, ref_codes, chrom_begin, read_codes, stride, lengths, q, w, sampled,
                    band, pct, mode, strands, mask, threads, with_threads_arg=True)


def _map(lib, name, b, ref_codes, chrom_begin, read_codes, stride, lengths, q, w, sampled, band, pct, mode, strands,
         mask, threads, with_threads_arg=True):
    ref_codes = np.ascontiguousarray(ref_codes, dtype=np.uint8)
    cb = np.ascontiguousarray(chrom_begin, dtype=np.uint64)
    read_codes, lengths = _reads_args(read_codes, stride, lengths)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    h = P()
    stats = np.zeros(9, dtype=np.uint64)  # 4 counts + 5 stage nanoseconds
    f = getattr(lib, name)
    f.argtypes = [P, P, C.c_uint32, P, P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32,
                  C.c_uint32, C.c_int, C.c_int, C.c_uint32, C.POINTER(P), P]
    b.check(f(_p(ref_codes), _p(cb), cb.size - 1, _p(m), _p(read_codes), stride, _p(lengths), lengths.size, q, w,
              int(sampled), band, pct, mode, strands, threads, C.byref(h), _p(stats)))
    hits = b.take(h, HIT_DTYPE)
    st = dict(zip(("raw_candidates", "unique_candidates", "validated", "hits"), stats[:4].tolist()))
    st["stage_seconds"] = dict(zip(("index", "filter", "sort_unique", "validate", "strata"),
                                   (round(float(x) / 1e9, 4) for x in stats[4:])))
    return hits, st


class RefShim:
    """The reference's own code behind a C ABI (oracle/_ref, built from /root/reference)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: build it with `make -C oracle` where /root/reference exists")
        self.lib = C.CDLL(path)
        self.b = _Buffers(self.lib, "ref_")

    def build_index(self, codes, stride, lengths, q, w=32, sampled=False, threads=1):
        codes, lengths = _reads_args(codes, stride, lengths)
        hs = [P() for _ in range(4)]
        f = self.lib.ref_build_index
        f.argtypes = [P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32] + [C.POINTER(P)] * 4
        self.b.check(f(_p(codes), stride, _p(lengths), lengths.size, q, w, int(sampled), threads,
                       *[C.byref(h) for h in hs]))
        wd = np.uint32 if w == 32 else np.uint64
        return (self.b.take(hs[0], wd), self.b.take(hs[1], np.uint32), self.b.take(hs[2], np.uint32),
                self.b.take(hs[3], np.uint32))

    def build_index_timed(self, codes, stride, lengths, q, threads):
        codes, lengths = _reads_args(codes, stride, lengths)
        sec, dist = C.c_double(), C.c_uint64()
        f = self.lib.ref_build_index_timed
        f.argtypes = [P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_double),
                      C.POINTER(C.c_uint64)]
        self.b.check(f(_p(codes), stride, _p(lengths), lengths.size, q, threads, C.byref(sec), C.byref(dist)))
        return sec.value, dist.value

    def filter_hits(self, ref_positions, ref_codes, read_codes, stride, lengths, q):
        pos = np.ascontiguousarray(ref_positions, dtype=np.uint32)
        cod = np.ascontiguousarray(ref_codes, dtype=np.uint32)
        read_codes, lengths = _reads_args(read_codes, stride, lengths)
        h = P()
        f = self.lib.ref_filter_hits
        f.argtypes = [P, P, C.c_uint64, P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.POINTER(P)]
        self.b.check(f(_p(pos), _p(cod), pos.size, _p(read_codes), stride, _p(lengths), lengths.size, q, C.byref(h)))
        return self.b.take(h, REFHIT_DTYPE)

    def _pair(self, name, read, window, extra):
        read = np.ascontiguousarray(read, dtype=np.uint8)
        window = np.ascontiguousarray(window, dtype=np.uint8)
        f = getattr(self.lib, name)
        f.restype = C.c_int
        f.argtypes = [P, C.c_uint32, P, C.c_uint32] + [C.c_uint32] * len(extra)
        return f(_p(read), read.size, _p(window), window.size, *extra)

    def banded_distance(self, read, window, band):
        return self._pair("ref_banded_distance", read, window, [band])

    def semiglobal_distance(self, read, window):
        return self._pair("ref_semiglobal_distance", read, window, [])

    def anchored_start_distance(self, read, window, start):
        return self._pair("ref_anchored_start_distance", read, window, [start])

    def encode_qgram(self, window):
        w = np.ascontiguousarray(window, dtype=np.uint8)
        out = C.c_uint32()
        f = self.lib.ref_encode_qgram
        f.argtypes = [P, C.c_uint32, C.POINTER(C.c_uint32)]
        self.b.check(f(_p(w), w.size, C.byref(out)))
        return out.value

    def pack_reads(self, reads, stride, q, seed):
        joined = b"".join(r.encode() + b"\0" for r in reads)
        buf = C.create_string_buffer(joined, len(joined) + 1)
        hc, hv = P(), P()
        f = self.lib.ref_pack_reads
        f.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(P), C.POINTER(P)]
        self.b.check(f(buf, len(reads), stride, q, seed, C.byref(hc), C.byref(hv)))
        return self.b.take(hc, np.uint8), self.b.take(hv, np.uint32)

    def exclusive_scan(self, values, threads=1):
        v = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.zeros(v.size, dtype=np.uint32)
        tot = C.c_uint32()
        f = self.lib.ref_exclusive_scan
        f.argtypes = [P, C.c_uint64, C.c_uint32, P, C.POINTER(C.c_uint32)]
        self.b.check(f(_p(v), v.size, threads, _p(out), C.byref(tot)))
        return out, tot.value

    def index_size_words(self, q, text_len, width):
        a, b, r = C.c_uint64(), C.c_uint64(), C.c_double()
        f = self.lib.ref_index_size_words
        f.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                      C.POINTER(C.c_double)]
        f(q, text_len, width, C.byref(a), C.byref(b), C.byref(r))
        return a.value, b.value, r.value

    def map(self, ref_codes, chrom_begin, read_codes, stride, lengths, q=16, w=32, sampled=False, band=32, pct=80,
            mode=0, strands=3, mask=None, threads=0):
        return _map(self.lib, "ref_map", self.b, ref_codes, chrom_begin, read_codes, stride, lengths, q, w, sampled,
                    band, pct, mode, strands, mask, threads)


def sort_intervals(S1, O):
    """Normalise O: sort positions inside every S' interval (test_parallel.cpp:121-122)."""
    O = O.copy()
    for b in range(S1.size - 1):
        lo, hi = int(S1[b]), int(S1[b + 1])
        if hi - lo > 1:
            O[lo:hi] = np.sort(O[lo:hi])
    return O


def rc_codes(codes):
    return (3 - np.asarray(codes, dtype=np.uint8)[::-1]).astype(np.uint8)


def repeat_mask(ref_codes, chrom_begin, q, threshold):
    """SPEC.md:302 restated in numpy: 1 for every position whose forward
    q-gram occurs more than `threshold` times among its chromosome's windows."""
    ref_codes = np.asarray(ref_codes, dtype=np.uint8)
    mask = np.zeros(ref_codes.size, np.uint8)
    for c in range(len(chrom_begin) - 1):
        b, e = int(chrom_begin[c]), int(chrom_begin[c + 1])
        if e - b < q:
            continue
        code = np.zeros(e - b - q + 1, np.uint64)
        for t in range(q):
            code = (code << np.uint64(2)) | ref_codes[b + t:e - q + 1 + t].astype(np.uint64)
        _, inv, cnt = np.unique(code, return_inverse=True, return_counts=True)
        mask[b:b + code.size] = cnt[inv] > threshold
    return mask


def cigar_string(ops, n_ops):
    """BAM-style ops (length << 4 | op, M=0 I=1 D=2) -> CIGAR text."""
    return "".join(f"{int(x) >> 4}{'MID'[int(x) & 15]}" for x in ops[:n_ops])

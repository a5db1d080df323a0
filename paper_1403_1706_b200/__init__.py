"""paper_1403_1706_b200 -- B200-native (sm_100a) PEANUT read-mapping hot path.

Python mirror of the reference's qgmap operator surface over the C ABI in
include/qgm_c.h (libqgm_b200.so, built in-tree by `make`). Names and argument
meaning follow the reference (proj/include/qgmap/{seq,qgroup_index}.hpp) and
SPEC.md for the spec-only stages:

    Context                      one CUDA device + stream (qgm_ctx)
    Reads.from_codes / upload    PackedReadText (seq.hpp:98-140)
    Index.build                  build_qgroup_index<W> (qgroup_index.hpp:124-180)
      .sample / .normalize       sample_group_starts (:185-196) / per-interval sort
      .occupancy .group_starts   the four arrays (:42-45)
      .occ_starts .positions
      .index_pair(codes)         Indexpair (:50-57)
    Reference.from_codes         ReferenceIndex sequences
    Context.filter               Alg. 2 filtration
    Context.validate             myers_banded / validate_hits
    Context.map / map_host       run_map core

There is no CPU fallback: if the shared library or a CUDA device is missing,
every entry point raises. Errors map like the reference: QGM_ERR_INPUT ->
InputError (qgmap::input_error), QGM_ERR_INTERNAL -> LogicError
(std::logic_error), QGM_ERR_CUDA -> CudaError.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QGM_LIB") or os.path.join(_HERE, "libqgm_b200.so")
SYNTH_PATH = os.path.join(_HERE, "libqgm_synth.so")

MODE_BEST_STRATUM = 0
MODE_ALL = 1
FILTER_FULL = 0
FILTER_RUN_START = 1
FILTER_JOIN = 2  # flag: bucket-ordered join with the reference q-group index (join.cu)
FILTER_STREAM = 4  # flag: streaming kernel (filter.cu); neither flag = the join below 2^32 padded bases
STAGES = ("reads", "index", "filter", "sort_unique", "validate", "strata", "d2h", "other")

CANDIDATE_DTYPE = np.dtype([("diagonal", "<i8"), ("read_id", "<u4"), ("chrom", "<u4"),
                            ("strand", "<u4"), ("reserved", "<u4")])
VALIDATED_DTYPE = np.dtype([("edits", "<i4"), ("start", "<u4"), ("ref_start", "<u4"), ("kept", "u1"),
                            ("in_range", "u1"), ("r0", "u1"), ("r1", "u1"), ("r2", "<u4")])
HIT_DTYPE = np.dtype([("read_id", "<u4"), ("chrom", "<u4"), ("ref_start", "<u4"), ("edits", "<u2"),
                      ("strand", "u1"), ("reserved", "u1")])
CIGAR_DTYPE = np.dtype([("ref_start", "<u4"), ("n_ops", "<u2"), ("edits", "<u2")])
assert CANDIDATE_DTYPE.itemsize == 24 and VALIDATED_DTYPE.itemsize == 20 and HIT_DTYPE.itemsize == 16


class QgmError(RuntimeError):
    pass


class InputError(QgmError, ValueError):
    """qgmap::input_error (seq.hpp:13-16)."""


class LogicError(QgmError):
    """std::logic_error (parallel.hpp:176,181)."""


class CudaError(QgmError):
    pass


class MapParams(C.Structure):
    _fields_ = [("q", C.c_uint32), ("group_width", C.c_uint32), ("sampled", C.c_uint32),
                ("band_width", C.c_uint32), ("pct_identity", C.c_uint32), ("mode", C.c_uint32),
                ("strands", C.c_uint32), ("reserved", C.c_uint32)]


class IndexInfo(C.Structure):
    _fields_ = [("q", C.c_uint32), ("group_width", C.c_uint32), ("sampled", C.c_uint32), ("reserved", C.c_uint32),
                ("group_count", C.c_uint64), ("group_starts_len", C.c_uint64), ("distinct", C.c_uint64),
                ("occurrences", C.c_uint64)]


class MapStats(C.Structure):
    _fields_ = [("raw_candidates", C.c_uint64), ("unique_candidates", C.c_uint64), ("validated", C.c_uint64),
                ("hits", C.c_uint64), ("index_distinct", C.c_uint64), ("index_occurrences", C.c_uint64),
                ("lookups_hit", C.c_uint64), ("occurrences", C.c_uint64)]


class Batch(C.Structure):
    """qgm_batch (include/qgm_c.h): one read buffer of qgm_map_host_batches."""
    _fields_ = [("reads2bit", C.c_void_p), ("lengths", C.c_void_p), ("n_reads", C.c_uint32), ("stride", C.c_uint32),
                ("out", C.c_void_p), ("cap", C.c_uint64), ("n_out", C.c_uint64), ("stats", MapStats),
                ("layout", C.c_uint32), ("reserved", C.c_uint32)]


READS_PADDED, READS_DENSE = 0, 1


# Every symbol include/qgm_c.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "qgm_ctx_create", "qgm_ctx_set_stream", "qgm_ctx_stream", "qgm_ctx_destroy", "qgm_last_error",
    "qgm_ctx_synchronize", "qgm_ctx_profile", "qgm_ctx_stage_times", "qgm_ctx_kernel_times", "qgm_ctx_launches", "qgm_pack_codes",
    "qgm_pack_reads", "qgm_reads_upload", "qgm_reads_from_device", "qgm_reads_destroy", "qgm_index_build",
    "qgm_index_sample", "qgm_index_normalize", "qgm_index_info_get", "qgm_index_download", "qgm_index_lookup",
    "qgm_index_destroy", "qgm_ref_upload", "qgm_ref_prepare", "qgm_ref_mask_repeats", "qgm_ref_mask_download",
    "qgm_ref_positions", "qgm_hits_ranks", "qgm_hits_cigar", "qgm_cigar_records",
    "qgm_ref_destroy", "qgm_filter", "qgm_cands_count",
    "qgm_cands_download", "qgm_cands_unique", "qgm_cands_destroy", "qgm_validate", "qgm_map", "qgm_hits_count",
    "qgm_hits_stats", "qgm_hits_download", "qgm_hits_destroy", "qgm_map_host", "qgm_map_host_batches",
    "qgm_exclusive_scan_u32",
)

_lib = None
_synth = None
P = C.c_void_p


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build_stamp() -> str:
    """Identity of the library build for matching ncu evidence to it: the
    sha256 of its CUDA sources and the Makefile (compiler flags) -- nvcc's
    output is not byte-reproducible across rebuilds of the same sources. A
    QGM_LIB override (an experiment build) is stamped by its bytes."""
    import glob
    import hashlib
    h = hashlib.sha256()
    if os.environ.get("QGM_LIB"):
        with open(LIB_PATH, "rb") as f:
            h.update(f.read())
        return h.hexdigest()[:16]
    root = os.path.dirname(_HERE)
    files = sorted(glob.glob(os.path.join(_HERE, "csrc", "*.cu")) + glob.glob(os.path.join(_HERE, "csrc", "*.cuh")) +
                   glob.glob(os.path.join(_HERE, "csrc", "*.hpp")) + [os.path.join(root, "Makefile")])
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def load_library(path: str = LIB_PATH):
    """Load libqgm_b200.so and declare the C ABI. Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `make` (or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
    sig = {
        "qgm_ctx_create": (i32, [i32, C.POINTER(P)]),
        "qgm_ctx_set_stream": (i32, [P, P]),
        "qgm_ctx_stream": (P, [P]),
        "qgm_ctx_destroy": (None, [P]),
        "qgm_last_error": (C.c_char_p, [P]),
        "qgm_ctx_synchronize": (i32, [P]),
        "qgm_ctx_profile": (i32, [P, i32]),
        "qgm_ctx_stage_times": (i32, [P, P, i32, i32]),
        "qgm_ctx_kernel_times": (i32, [P, C.c_char_p, u64, i32]),
        "qgm_ctx_launches": (u64, [P, i32]),
        "qgm_pack_codes": (i32, [P, u64, P]),
        "qgm_pack_reads": (i32, [P, u32, u32, P]),
        "qgm_reads_upload": (i32, [P, P, P, u32, u32, C.POINTER(P)]),
        "qgm_reads_from_device": (i32, [P, P, P, u32, u32, C.POINTER(P)]),
        "qgm_reads_destroy": (None, [P]),
        "qgm_index_build": (i32, [P, P, u32, u32, i32, C.POINTER(P)]),
        "qgm_index_sample": (i32, [P, P, C.POINTER(P)]),
        "qgm_index_normalize": (i32, [P, P]),
        "qgm_index_info_get": (i32, [P, C.POINTER(IndexInfo)]),
        "qgm_index_download": (i32, [P, P, P, P, P, P]),
        "qgm_index_lookup": (i32, [P, P, P, u64, P, P]),
        "qgm_index_destroy": (None, [P]),
        "qgm_ref_upload": (i32, [P, P, P, u32, P, C.POINTER(P)]),
        "qgm_ref_prepare": (i32, [P, P, u32]),
        "qgm_ref_mask_repeats": (i32, [P, P, u32, u64]),
        "qgm_ref_mask_download": (i32, [P, P, P]),
        "qgm_ref_positions": (i32, [P, P, u32, C.POINTER(u64)]),
        "qgm_hits_ranks": (i32, [P, P, P]),
        "qgm_hits_cigar": (i32, [P, P, P, P, u32, u32, P, P]),
        "qgm_cigar_records": (i32, [P, P, P, P, u64, u32, u32, P, P]),
        "qgm_ref_destroy": (None, [P]),
        "qgm_filter": (i32, [P, P, P, P, i32, i32, C.POINTER(P)]),
        "qgm_cands_count": (i32, [P, C.POINTER(u64)]),
        "qgm_cands_download": (i32, [P, P, P]),
        "qgm_cands_unique": (i32, [P, P]),
        "qgm_cands_destroy": (None, [P]),
        "qgm_validate": (i32, [P, P, P, P, u64, u32, u32, P]),
        "qgm_map": (i32, [P, P, P, C.POINTER(MapParams), C.POINTER(P)]),
        "qgm_hits_count": (i32, [P, C.POINTER(u64)]),
        "qgm_hits_stats": (i32, [P, C.POINTER(MapStats)]),
        "qgm_hits_download": (i32, [P, P, P]),
        "qgm_hits_destroy": (None, [P]),
        "qgm_map_host": (i32, [P, P, P, u32, u32, P, C.POINTER(MapParams), P, u64, C.POINTER(u64),
                               C.POINTER(MapStats)]),
        "qgm_map_host_batches": (i32, [P, P, u32, P, C.POINTER(MapParams)]),
        "qgm_exclusive_scan_u32": (i32, [P, P, u64, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def load_synth(path: str = SYNTH_PATH):
    global _synth
    if _synth is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `make`")
        s = C.CDLL(path)
        s.qgs_random_reference.argtypes = [C.c_uint64, C.c_uint64, P]
        s.qgs_repetitive_reference.argtypes = [C.c_uint64, C.c_uint64, P]
        s.qgs_simulate_reads.argtypes = [C.c_uint64, P, P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                         C.c_uint32, P, P, P, P, P]
        s.qgs_pack.argtypes = [P, C.c_uint64, P]
        s.qgs_pack_reads.argtypes = [P, C.c_uint32, C.c_uint32, P]
        _synth = s
    return _synth


# ----------------------------------------------------------------- host codec
def mapping_quality(rank, p_size: int):
    """mapping_quality: min{-10 log10((R-1)/|P|), 255}, R=1 ->
    255, rounded half up, floored at 0 (host floating point; vectorised)."""
    r = np.asarray(rank, dtype=np.float64)
    with np.errstate(divide="ignore"):
        q = -10.0 * np.log10(np.maximum(r - 1.0, 0.0) / max(p_size, 1))
    q = np.floor(np.minimum(q, 255.0) + 0.5)
    return np.where(r <= 1, 255, np.maximum(q, 0)).astype(np.uint8)


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """1-byte codes (0..3) -> 2-bit MSB-first uint64 words (qgm_c.h layout)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    words = np.zeros((codes.size + 31) // 32 + 1, dtype=np.uint64)
    load_synth().qgs_pack(_ptr(codes), codes.size, _ptr(words))
    return words


def pack_read_codes(codes: np.ndarray, stride: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n = codes.size // stride if stride else 0
    W = (stride + 31) // 32
    words = np.zeros(max(n * W, 1), dtype=np.uint64)
    if n:
        load_synth().qgs_pack_reads(_ptr(codes), stride, n, _ptr(words))
    return words


def random_reference(seed: int, length: int) -> np.ndarray:
    out = np.empty(length, dtype=np.uint8)
    load_synth().qgs_random_reference(seed, length, _ptr(out))
    return out


def repetitive_reference(seed: int, length: int) -> np.ndarray:
    out = np.empty(length, dtype=np.uint8)
    load_synth().qgs_repetitive_reference(seed, length, _ptr(out))
    return out


def simulate_reads(seed, ref_codes, chrom_begin, n_reads, length, err, stride=None):
    """Returns (codes[n_reads*stride], lengths, truth_chrom, truth_pos, truth_strand)."""
    stride = stride or length
    ref_codes = np.ascontiguousarray(ref_codes, dtype=np.uint8)
    cb = np.ascontiguousarray(chrom_begin, dtype=np.uint64)
    codes = np.zeros(n_reads * stride, dtype=np.uint8)
    lengths = np.zeros(n_reads, dtype=np.uint32)
    tc = np.zeros(n_reads, dtype=np.uint32)
    tp = np.zeros(n_reads, dtype=np.uint64)
    ts = np.zeros(n_reads, dtype=np.uint8)
    rc = load_synth().qgs_simulate_reads(seed, _ptr(ref_codes), _ptr(cb), cb.size - 1, n_reads, length, err, stride,
                                         _ptr(codes), _ptr(lengths), _ptr(tc), _ptr(tp), _ptr(ts))
    if rc:
        raise InputError("simulate_reads: bad arguments")
    return codes, lengths, tc, tp, ts


# ----------------------------------------------------------------- objects
class Context:
    """One device + stream (qgm_ctx). All objects must be released before it."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load_library()
        self._children = weakref.WeakSet()  # Reads / Reference / Index handles owned by this context
        h = P()
        self._check(self.lib.qgm_ctx_create(device, C.byref(h)), None)
        self.h = h
        if stream is not None:
            self._check(self.lib.qgm_ctx_set_stream(self.h, P(stream)))

    def _adopt(self, obj):
        self._children.add(obj)
        return obj

    def _check(self, rc, h=...):
        if rc == 0:
            return
        msg = self.lib.qgm_last_error(self.h if h is ... else h)
        msg = msg.decode() if msg else f"error {rc}"
        raise {1: InputError, 2: LogicError, 3: CudaError}.get(rc, QgmError)(msg)

    def close(self):
        """Destroy the context; every live child handle is released first
        (a child's native destroy touches its context)."""
        if getattr(self, "h", None):
            for child in list(getattr(self, "_children", ())):
                child.close()
            self.lib.qgm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        self._check(self.lib.qgm_ctx_synchronize(self.h))

    def set_stream(self, stream: int | None):
        self._check(self.lib.qgm_ctx_set_stream(self.h, P(stream) if stream else None))

    def profile(self, enable=True):
        self._check(self.lib.qgm_ctx_profile(self.h, int(enable)))

    def stage_times(self, reset=True, host=False) -> dict:
        """GPU (CUDA-event) ms per stage; with host=True also the host wall ms."""
        ms = np.zeros(2 * len(STAGES), dtype=np.float64)
        self._check(self.lib.qgm_ctx_stage_times(self.h, _ptr(ms), ms.size, int(reset)))
        out = dict(zip(STAGES, ms[:len(STAGES)].tolist()))
        if host:
            out.update({"host_" + k: v for k, v in zip(STAGES, ms[len(STAGES):].tolist())})
        return out

    def kernel_times(self, reset=True) -> dict:
        """{kernel: (total_ms, launches)} for the timed hot kernels (profile mode)."""
        buf = C.create_string_buffer(1 << 16)
        self._check(self.lib.qgm_ctx_kernel_times(self.h, buf, len(buf), int(reset)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, ms, n = line.split("\t")
            out[name] = (float(ms), int(n))
        return out

    def launches(self, reset=False) -> int:
        return int(self.lib.qgm_ctx_launches(self.h, int(reset)))

    # --- stage entry points
    def filter(self, index, reads, ref, strands=3, mode=FILTER_FULL, unique=False) -> np.ndarray:
        h = P()
        self._check(self.lib.qgm_filter(self.h, index.h, reads.h, ref.h, strands, mode, C.byref(h)))
        try:
            if unique:
                self._check(self.lib.qgm_cands_unique(self.h, h))
            n = C.c_uint64()
            self._check(self.lib.qgm_cands_count(h, C.byref(n)))
            out = np.zeros(n.value, dtype=CANDIDATE_DTYPE)
            self._check(self.lib.qgm_cands_download(self.h, h, _ptr(out)))
            return out
        finally:
            self.lib.qgm_cands_destroy(h)

    def validate(self, reads, ref, cands: np.ndarray, band_width=32, pct_identity=80) -> np.ndarray:
        cands = np.ascontiguousarray(cands, dtype=CANDIDATE_DTYPE)
        out = np.zeros(cands.size, dtype=VALIDATED_DTYPE)
        self._check(self.lib.qgm_validate(self.h, reads.h, ref.h, _ptr(cands), cands.size, band_width,
                                          pct_identity, _ptr(out)))
        return out

    def map(self, reads, ref, params: MapParams | None = None, ranks: bool = False, cigars: bool = False, **kw):
        """Returns (hits[HIT_DTYPE], stats dict) -- with ranks=True also the
        hit_rank of every record, with cigars=True also
        (ops, info) of traceback_cigar computed from the device-resident hits
        (SPEC.md:476-483): (hits, stats[, ranks][, (ops, info)])."""
        p = params or make_params(**kw)
        h = P()
        self._check(self.lib.qgm_map(self.h, reads.h, ref.h, C.byref(p), C.byref(h)))
        try:
            n = C.c_uint64()
            self._check(self.lib.qgm_hits_count(h, C.byref(n)))
            st = MapStats()
            self._check(self.lib.qgm_hits_stats(h, C.byref(st)))
            out = np.zeros(n.value, dtype=HIT_DTYPE)
            self._check(self.lib.qgm_hits_download(self.h, h, _ptr(out)))
            stats = {f: getattr(st, f) for f, _ in MapStats._fields_}
            res = [out, stats]
            if ranks:
                r = np.zeros(max(n.value, 1), dtype=np.uint32)
                self._check(self.lib.qgm_hits_ranks(self.h, h, _ptr(r)))
                res.append(r[: n.value])
            if cigars:
                # like map.hpp run_cigar: a small record first, one retry at
                # the size the longest record needs
                band = p.band_width
                max_ops = 2 * band + 16
                info = np.zeros(n.value, CIGAR_DTYPE)
                ops = np.zeros((n.value, max_ops), np.uint32)
                rc = self.lib.qgm_hits_cigar(self.h, h, reads.h, ref.h, band, max_ops, _ptr(ops), _ptr(info))
                if rc == 1 and n.value and int(info["n_ops"].max()) > max_ops:
                    max_ops = int(info["n_ops"].max())
                    ops = np.zeros((n.value, max_ops), np.uint32)
                    rc = self.lib.qgm_hits_cigar(self.h, h, reads.h, ref.h, band, max_ops, _ptr(ops), _ptr(info))
                self._check(rc)
                res.append((ops, info))
            return tuple(res)
        finally:
            self.lib.qgm_hits_destroy(h)

    def cigar(self, reads, ref, hits: np.ndarray, band_width: int = 32, max_ops: int | None = None):
        """traceback_cigar (DESIGN.md section 2 item 9) of hit
        records on the device: (ops[n, max_ops] u32 BAM-style, info[CIGAR_DTYPE]).
        max_ops defaults to 2 * (stride + band_width) + 1, enough for any record."""
        hits = np.ascontiguousarray(hits, dtype=HIT_DTYPE)
        if max_ops is None:
            max_ops = 2 * (reads.stride + band_width) + 1
        ops = np.zeros((hits.size, max_ops), np.uint32)
        info = np.zeros(hits.size, CIGAR_DTYPE)
        self._check(self.lib.qgm_cigar_records(self.h, reads.h, ref.h, _ptr(hits), hits.size, band_width, max_ops,
                                               _ptr(ops), _ptr(info)))
        return ops, info

    def map_host(self, words: np.ndarray, lengths: np.ndarray, stride: int, ref, params=None, out=None, **kw):
        """e2e entry: host reads in, host hits out (qgm_map_host)."""
        p = params or make_params(**kw)
        lengths = np.ascontiguousarray(lengths, dtype=np.uint32)
        if out is None:
            out = np.zeros(max(64, lengths.size * 4), dtype=HIT_DTYPE)
        n = C.c_uint64()
        st = MapStats()
        rc = self.lib.qgm_map_host(self.h, _ptr(words), _ptr(lengths), lengths.size, stride, ref.h, C.byref(p),
                                   _ptr(out), out.size, C.byref(n), C.byref(st))
        if rc == 1 and n.value > out.size:
            out = np.zeros(n.value, dtype=HIT_DTYPE)
            rc = self.lib.qgm_map_host(self.h, _ptr(words), _ptr(lengths), lengths.size, stride, ref.h, C.byref(p),
                                       _ptr(out), out.size, C.byref(n), C.byref(st))
        self._check(rc)
        return out[: n.value], {f: getattr(st, f) for f, _ in MapStats._fields_}

    def map_host_batches(self, batches, ref, params=None, **kw):
        """Streamed e2e entry (qgm_map_host_batches): `batches` is a list of
        (words, lengths, stride[, layout, n_reads]) host arrays -- layout
        READS_DENSE takes a qgm_pack_codes stream, lengths None means every
        read has length `stride`; returns [(hits, stats), ...].
        Pinned host arrays let the copies overlap the mapping."""
        p = params or make_params(**kw)
        arr = (Batch * len(batches))()
        keep = []
        for i, bt in enumerate(batches):
            words, lengths, stride = bt[:3]
            layout = bt[3] if len(bt) > 3 else READS_PADDED
            n_reads = bt[4] if len(bt) > 4 else np.asarray(lengths).size
            lengths = None if lengths is None else np.ascontiguousarray(lengths, dtype=np.uint32)
            out = np.zeros(max(64, n_reads * 4), dtype=HIT_DTYPE)
            keep.append((words, lengths, out))
            arr[i] = Batch(_ptr(words), _ptr(lengths) if lengths is not None else None, n_reads, stride, _ptr(out),
                           out.size, 0, MapStats(), layout, 0)
        rc = self.lib.qgm_map_host_batches(self.h, arr, len(batches), ref.h, C.byref(p))
        if rc == 1 and any(arr[i].n_out > arr[i].cap for i in range(len(batches))):
            for i, (words, lengths, out) in enumerate(keep):
                if arr[i].n_out > arr[i].cap:
                    out = np.zeros(arr[i].n_out, dtype=HIT_DTYPE)
                    keep[i] = (words, lengths, out)
                    arr[i].out, arr[i].cap = _ptr(out), out.size
            rc = self.lib.qgm_map_host_batches(self.h, arr, len(batches), ref.h, C.byref(p))
        self._check(rc)
        return [(keep[i][2][: arr[i].n_out], {f: getattr(arr[i].stats, f) for f, _ in MapStats._fields_})
                for i in range(len(batches))]

    def exclusive_scan(self, values: np.ndarray):
        """par::exclusive_scan (parallel.hpp:116-121) on the device: (sums, total)."""
        v = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.zeros(v.size, dtype=np.uint32)
        tot = C.c_uint32()
        self._check(self.lib.qgm_exclusive_scan_u32(self.h, _ptr(v), v.size, _ptr(out), C.byref(tot)))
        return out, tot.value


def make_params(q=16, group_width=32, sampled=False, band_width=32, pct_identity=80, mode=MODE_BEST_STRATUM,
                strands=3) -> MapParams:
    return MapParams(q, group_width, int(sampled), band_width, pct_identity, mode, strands, 0)


class Reads:
    """A read buffer on the device (PackedReadText, seq.hpp:98-115)."""

    def __init__(self, ctx: Context, words: np.ndarray, lengths: np.ndarray, stride: int):
        self.ctx = ctx
        lengths = np.ascontiguousarray(lengths, dtype=np.uint32)
        words = np.ascontiguousarray(words, dtype=np.uint64)
        self.n, self.stride = lengths.size, stride
        h = P()
        ctx._check(ctx.lib.qgm_reads_upload(ctx.h, _ptr(words), _ptr(lengths), lengths.size, stride, C.byref(h)))
        self.h = h
        ctx._adopt(self)

    @classmethod
    def from_codes(cls, ctx, codes: np.ndarray, lengths: np.ndarray, stride: int):
        return cls(ctx, pack_read_codes(codes, stride), lengths, stride)

    def close(self):
        if getattr(self, "h", None):
            if getattr(self.ctx, "h", None):  # the context destroys nothing twice
                self.ctx.lib.qgm_reads_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Reference:
    """Reference sequences on the device (concatenated chromosomes, optional repeat mask)."""

    def __init__(self, ctx: Context, words, chrom_begin, mask_bits: np.ndarray | None = None):
        """words: the 2-bit words as a host array, or an int device pointer
        (e.g. the broadcast copy of a multi-GPU run; qgm_ref_upload takes
        either)."""
        self.ctx = ctx
        cb = np.ascontiguousarray(chrom_begin, dtype=np.uint64)
        self.chrom_begin = cb
        if isinstance(words, int):
            wp = P(words)
        else:
            words = np.ascontiguousarray(words, dtype=np.uint64)
            wp = _ptr(words)
        mb = None if mask_bits is None else np.ascontiguousarray(mask_bits, dtype=np.uint64)
        h = P()
        ctx._check(ctx.lib.qgm_ref_upload(ctx.h, wp, _ptr(cb), cb.size - 1, _ptr(mb), C.byref(h)))
        self.h = h
        ctx._adopt(self)

    @classmethod
    def from_codes(cls, ctx, codes: np.ndarray, chrom_begin, mask: np.ndarray | None = None):
        mb = None
        if mask is not None:
            m = np.ascontiguousarray(mask, dtype=np.uint8).astype(bool)
            padded = np.zeros((m.size + 63) // 64 * 64, dtype=bool)
            padded[: m.size] = m
            mb = np.packbits(padded, bitorder="little").view(np.uint64).copy() \
                if padded.size else np.zeros(1, np.uint64)
        return cls(ctx, pack_codes(codes), chrom_begin, mb)

    def mask_repeats(self, q: int, threshold: int = 1000):
        """Repeat mask on the device: positions whose forward
        q-gram occurs more than `threshold` times in their chromosome leave P."""
        self.ctx._check(self.ctx.lib.qgm_ref_mask_repeats(self.ctx.h, self.h, q, threshold))
        return self

    def mask(self) -> np.ndarray:
        """The current mask as one uint8 per base (1 = not in P)."""
        total = int(self.chrom_begin[-1])
        words = np.zeros(max((total + 63) // 64, 1), np.uint64)
        self.ctx._check(self.ctx.lib.qgm_ref_mask_download(self.ctx.h, self.h, _ptr(words)))
        return np.unpackbits(words.view(np.uint8), bitorder="little")[:total]

    def positions(self, q: int) -> int:
        """|P| for q: reference positions in P (mapping_quality's P_size)."""
        v = C.c_uint64()
        self.ctx._check(self.ctx.lib.qgm_ref_positions(self.ctx.h, self.h, q, C.byref(v)))
        return v.value

    def prepare(self, q: int):
        """Build the reference-side q-group index for q (qgm_ref_prepare)."""
        self.ctx._check(self.ctx.lib.qgm_ref_prepare(self.ctx.h, self.h, q))
        return self

    def close(self):
        if getattr(self, "h", None):
            if getattr(self.ctx, "h", None):  # the context destroys nothing twice
                self.ctx.lib.qgm_ref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Index:
    """QGroupIndex<W> on the device (qgroup_index.hpp:28-104)."""

    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        ctx._adopt(self)
        info = IndexInfo()
        ctx._check(ctx.lib.qgm_index_info_get(h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in IndexInfo._fields_}
        self._arrays = None

    @classmethod
    def build(cls, ctx: Context, reads: Reads, q: int, group_width: int = 32, sampled: bool = False):
        h = P()
        ctx._check(ctx.lib.qgm_index_build(ctx.h, reads.h, q, group_width, int(sampled), C.byref(h)))
        return cls(ctx, h)

    def sample(self) -> "Index":
        h = P()
        self.ctx._check(self.ctx.lib.qgm_index_sample(self.ctx.h, self.h, C.byref(h)))
        return Index(self.ctx, h)

    def normalize(self):
        self.ctx._check(self.ctx.lib.qgm_index_normalize(self.ctx.h, self.h))
        self._arrays = None
        return self

    def arrays(self):
        if self._arrays is None:
            i = self.info
            wd = np.uint32 if i["group_width"] == 32 else np.uint64
            I = np.zeros(i["group_count"], dtype=wd)
            S = np.zeros(i["group_starts_len"], dtype=np.uint32)
            S1 = np.zeros(i["distinct"] + 1, dtype=np.uint32)
            O = np.zeros(i["occurrences"], dtype=np.uint32)
            self.ctx._check(self.ctx.lib.qgm_index_download(self.ctx.h, self.h, _ptr(I), _ptr(S), _ptr(S1), _ptr(O)))
            self._arrays = (I, S, S1, O)
        return self._arrays

    occupancy = property(lambda self: self.arrays()[0])
    group_starts = property(lambda self: self.arrays()[1])
    occ_starts = property(lambda self: self.arrays()[2])
    positions = property(lambda self: self.arrays()[3])

    def index_pair(self, codes):
        codes = np.ascontiguousarray(np.atleast_1d(codes), dtype=np.uint32)
        b = np.zeros(codes.size, dtype=np.uint32)
        e = np.zeros(codes.size, dtype=np.uint32)
        self.ctx._check(self.ctx.lib.qgm_index_lookup(self.ctx.h, self.h, _ptr(codes), codes.size, _ptr(b), _ptr(e)))
        return b, e

    def close(self):
        if getattr(self, "h", None):
            if getattr(self.ctx, "h", None):  # the context destroys nothing twice
                self.ctx.lib.qgm_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cigar_string(ops: np.ndarray, n_ops: int) -> str:
    """BAM-style ops (length << 4 | op, M=0 I=1 D=2) -> CIGAR text."""
    return "".join(f"{int(x) >> 4}{'MID'[int(x) & 15]}" for x in ops[:n_ops])

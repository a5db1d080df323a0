"""Reference-sharded mapping (PAPER.md:262,
"all steps are performed per chromosome").

Read sharding (sharding.py) replicates the reference, so every GPU streams the
whole reference index per batch: filtration does not shrink with G
(SURVEY 8(e)). Here the *reference* is split instead: every rank maps the
whole read batch against its share of the reference, then the ranks exchange
the per-read results -- the one real data exchange of this path:

  1. best-stratum only: all-reduce MIN of every read's smallest edit count
     (one int32 per read), after which a rank keeps only its hits at that
     minimum (the strata rule, applied across shards);
  2. all-to-all of the surviving 16-byte hit records to the rank that owns the
     read (contiguous read ranges, sharding.shard_range), which sorts them.

Exactness. A share is a set of pieces; a piece owns the chromosome-relative
ref_start range [own_begin, own_end) and carries the bases
[own_begin - 2B, own_end + n_max + 2B) of its chromosome (clipped to it). A
candidate whose ref_start s is owned has its validation window
[d - H, d - H + n + B - 1), d - H in (s - B, s], inside the piece, so its k
and start are those of the whole reference; a window that crosses a piece
cut gets sentinel bases, but then its ref_start lies outside the owned range
(more than B left of own_begin, or right of own_end) and the piece drops it.
The owned ranges partition every chromosome, so each hit comes from exactly
one piece and hit-level dedup (same ref_start -> same piece) stays local.
The repeat mask counts q-grams over whole chromosomes, so it is
computed once on the whole reference and sliced, never per piece.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import sharding


@dataclass(frozen=True)
class Piece:
    chrom: int      # chromosome of the whole reference
    own_begin: int  # owned ref_start range, chromosome-relative
    own_end: int
    begin: int      # bases carried, chromosome-relative
    end: int


def plan(chrom_begin, world_size: int, max_read_len: int, band: int) -> list[list[Piece]]:
    """Split the reference into world_size shares of near-equal owned length;
    chromosomes are cut where a share fills up. Returns the pieces of every
    rank (possibly none for tiny references)."""
    cb = np.asarray(chrom_begin, dtype=np.int64)
    lens = np.diff(cb)
    total = int(lens.sum())
    margin_l, margin_r = 2 * band, max_read_len + 2 * band
    shares: list[list[Piece]] = [[] for _ in range(world_size)]
    bounds = [sharding.shard_range(total, g, world_size) for g in range(world_size)]
    for g, (b, e) in enumerate(bounds):
        # global owned range [b, e) -> per-chromosome pieces
        for c in range(lens.size):
            lo, hi = max(b, int(cb[c])), min(e, int(cb[c + 1]))
            if lo >= hi:
                continue
            ob, oe = lo - int(cb[c]), hi - int(cb[c])
            shares[g].append(Piece(c, ob, oe, max(0, ob - margin_l), min(int(lens[c]), oe + margin_r)))
    return shares


def piece_reference(ref_codes, chrom_begin, pieces: list[Piece], mask=None):
    """Concatenated piece sequences as a reference of their own (one
    'chromosome' per piece): (codes, chrom_begin, mask or None)."""
    ref_codes = np.asarray(ref_codes, dtype=np.uint8)
    cb = np.asarray(chrom_begin, dtype=np.uint64)
    segs, msegs, out_cb = [], [], [0]
    for p in pieces:
        g0 = int(cb[p.chrom]) + p.begin
        segs.append(ref_codes[g0:g0 + p.end - p.begin])
        if mask is not None:
            msegs.append(np.asarray(mask, dtype=np.uint8)[g0:g0 + p.end - p.begin])
        out_cb.append(out_cb[-1] + p.end - p.begin)
    codes = np.concatenate(segs) if segs else np.zeros(0, np.uint8)
    m = (np.concatenate(msegs) if msegs else np.zeros(0, np.uint8)) if mask is not None else None
    return codes, np.array(out_cb, dtype=np.uint64), m


# ------------------------------------------------------------------ records
# The exchange runs on 16-byte hit records (qgm_hit, HIT_DTYPE) held in torch
# tensors on the rank's device: int32 view [n, 4] = read_id, chrom, ref_start,
# edits | strand << 16. Nothing crosses the host between the map and the
# sorted per-owner result; NCCL (or gloo for CPU tensors) carries the MIN
# all-reduce and the all-to-all.

def to_records(hits: np.ndarray, device="cpu"):
    """HIT_DTYPE numpy records -> int32 [n, 4] tensor on `device`."""
    import torch
    h = np.ascontiguousarray(hits)
    return torch.from_numpy(h.view(np.int32).reshape(-1, 4).copy()).to(device)


def from_records(rec) -> np.ndarray:
    """int32 [n, 4] tensor -> HIT_DTYPE numpy records."""
    from . import HIT_DTYPE
    return np.ascontiguousarray(rec.cpu().numpy()).view(HIT_DTYPE).reshape(-1)


def _u32(col):
    import torch
    return col.to(torch.int64) & 0xFFFFFFFF


def own_and_translate(rec, pieces: list[Piece]):
    """Keep the records whose ref_start a piece owns; piece-relative (chrom,
    ref_start) -> whole-reference chromosome coordinates. rec: int32 [n, 4]
    tensor (numpy HIT_DTYPE records are accepted and returned as numpy)."""
    import torch
    if isinstance(rec, np.ndarray):
        return from_records(own_and_translate(to_records(rec), pieces))
    if rec.shape[0] == 0 or not pieces:
        return rec[:0]
    dev = rec.device
    tab = torch.tensor([[p.begin, p.own_begin, p.own_end, p.chrom] for p in pieces], dtype=torch.int64, device=dev)
    pc = _u32(rec[:, 1])
    begin, ob, oe, chrom = (tab[:, i][pc] for i in range(4))
    pos = _u32(rec[:, 2]) + begin
    keep = (pos >= ob) & (pos < oe)
    out = rec[keep].clone()
    out[:, 1] = chrom[keep].to(torch.int32)
    out[:, 2] = pos[keep].to(torch.int32)  # < 2^32 (chromosomes < 2^32 - 1 bases), two's complement wraps
    return out


def sort_records(rec):
    """Sort by (read, chrom, ref_start, strand) -- the map's output order."""
    import torch
    if rec.shape[0] == 0:
        return rec
    key = (_u32(rec[:, 1]) << 33) | (_u32(rec[:, 2]) << 1) | ((rec[:, 3].to(torch.int64) >> 16) & 1)
    o1 = torch.sort(key, stable=True).indices
    rec = rec[o1]
    o2 = torch.sort(_u32(rec[:, 0]), stable=True).indices
    return rec[o2]


def best_stratum_filter(rec, n_reads: int, dist=None):
    """All-reduce MIN of every read's smallest edit count; keep the records at it."""
    import torch
    dev = rec.device
    big = torch.iinfo(torch.int32).max
    kmin = torch.full((n_reads,), big, dtype=torch.int32, device=dev)
    read = _u32(rec[:, 0])
    k = (rec[:, 3] & 0xFFFF).to(torch.int32)
    if rec.shape[0]:
        kmin.scatter_reduce_(0, read, k, reduce="amin")
    if dist is not None and dist.is_initialized():
        dist.all_reduce(kmin, op=dist.ReduceOp.MIN)
    return rec[k == kmin[read]] if rec.shape[0] else rec


def exchange_to_owners(rec, n_reads: int, dist=None):
    """All-to-all of the records to the rank owning the read's range
    (sharding.shard_range); returns this rank's reads' records sorted by
    (read, chrom, ref_start, strand)."""
    import torch
    if dist is None or not dist.is_initialized():
        return sort_records(rec)
    G = dist.get_world_size()
    dev = rec.device
    starts = torch.tensor([sharding.shard_range(n_reads, g, G)[0] for g in range(G)], dtype=torch.int64, device=dev)
    dest = torch.searchsorted(starts, _u32(rec[:, 0]), right=True) - 1
    order = torch.sort(dest, stable=True).indices
    send = rec[order].contiguous()
    send_counts = torch.bincount(dest, minlength=G).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts)
    rc = recv_counts.tolist()
    sc = send_counts.tolist()
    recv = torch.empty((int(sum(rc)), 4), dtype=torch.int32, device=dev)
    dist.all_to_all_single(recv, send, rc, sc)
    return sort_records(recv)


def combine(local, n_reads: int, mode: int, dist=None):
    """The exchange step: best-stratum MIN (mode 0) then records to the read
    owners. local: int32 [n, 4] tensor (or numpy HIT_DTYPE records, returned
    as numpy)."""
    if isinstance(local, np.ndarray):
        return from_records(combine(to_records(local), n_reads, mode, dist))
    rec = best_stratum_filter(local, n_reads, dist) if mode == 0 else local
    return exchange_to_owners(rec, n_reads, dist)


def map_ref_sharded(ctx, reads, ref_codes, chrom_begin, rank: int, world_size: int, params=None, mask=None,
                    dist=None, device="cpu", **kw):
    """One rank's part of a reference-sharded map of a whole read batch on the
    device: plan, upload this rank's pieces, map (all mode), download the hit
    records into a tensor on `device` (device to device for a CUDA device),
    keep the owned ones, exchange. Returns this rank's reads' records (int32
    [n, 4] tensor on `device`, whole-reference coordinates)."""
    import ctypes as C

    import torch

    from . import MapParams, MapStats, Reference, make_params

    p = params or make_params(**kw)
    shares = plan(chrom_begin, world_size, reads.stride, p.band_width)
    mine = shares[rank]
    local = torch.zeros((0, 4), dtype=torch.int32, device=device)
    if mine:
        codes, cb, m = piece_reference(ref_codes, chrom_begin, mine, mask)
        R = Reference.from_codes(ctx, codes, cb, mask=m)
        q = make_params(q=p.q, group_width=p.group_width, sampled=p.sampled, band_width=p.band_width,
                        pct_identity=p.pct_identity, mode=1, strands=p.strands)
        lib = ctx.lib
        h = C.c_void_p()
        ctx._check(lib.qgm_map(ctx.h, reads.h, R.h, C.byref(q), C.byref(h)))
        try:
            n = C.c_uint64()
            ctx._check(lib.qgm_hits_count(h, C.byref(n)))
            local = torch.empty((n.value, 4), dtype=torch.int32, device=device)
            if n.value:
                ctx._check(lib.qgm_hits_download(ctx.h, h, C.c_void_p(local.data_ptr())))
        finally:
            lib.qgm_hits_destroy(h)
        R.close()
        local = own_and_translate(local, mine)
    return combine(local, reads.n, p.mode, dist)

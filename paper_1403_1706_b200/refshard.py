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


def own_and_translate(hits: np.ndarray, pieces: list[Piece]) -> np.ndarray:
    """Keep the hits whose ref_start a piece owns; piece-relative (chrom,
    ref_start) -> whole-reference chromosome coordinates."""
    if hits.size == 0 or not pieces:
        return hits[:0]
    pc = hits["chrom"].astype(np.int64)
    begin = np.array([p.begin for p in pieces], np.int64)[pc]
    ob = np.array([p.own_begin for p in pieces], np.int64)[pc]
    oe = np.array([p.own_end for p in pieces], np.int64)[pc]
    chrom = np.array([p.chrom for p in pieces], np.int64)[pc]
    pos = hits["ref_start"].astype(np.int64) + begin
    keep = (pos >= ob) & (pos < oe)
    out = hits[keep].copy()
    out["chrom"] = chrom[keep]
    out["ref_start"] = pos[keep]
    return out


def _sorted(h: np.ndarray) -> np.ndarray:
    return h[np.lexsort((h["strand"], h["ref_start"], h["chrom"], h["read_id"]))] if h.size else h


def best_stratum_filter(hits: np.ndarray, n_reads: int, dist=None, device="cpu") -> np.ndarray:
    """All-reduce MIN of every read's smallest edit count; keep the hits at it."""
    import torch

    kmin = np.full(n_reads, np.iinfo(np.int32).max, np.int32)
    if hits.size:
        np.minimum.at(kmin, hits["read_id"].astype(np.int64), hits["edits"].astype(np.int32))
    if dist is not None and dist.is_initialized():
        t = torch.from_numpy(kmin).to(device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        kmin = t.cpu().numpy()
    return hits[hits["edits"].astype(np.int32) == kmin[hits["read_id"].astype(np.int64)]] if hits.size else hits


def exchange_to_owners(hits: np.ndarray, n_reads: int, dist=None, device="cpu") -> np.ndarray:
    """All-to-all of hit records to the rank owning the read's range; the
    result is this rank's reads' hits sorted by (read, chrom, ref_start,
    strand)."""
    import torch

    if dist is None or not dist.is_initialized():
        return _sorted(hits)
    G, me = dist.get_world_size(), dist.get_rank()
    starts = np.array([sharding.shard_range(n_reads, g, G)[0] for g in range(G)] + [n_reads], np.int64)
    dest = np.searchsorted(starts, hits["read_id"].astype(np.int64), side="right") - 1
    order = np.argsort(dest, kind="stable")
    send = np.ascontiguousarray(hits[order])
    send_counts = np.bincount(dest, minlength=G).astype(np.int64)
    sc = torch.from_numpy(send_counts).to(device)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc)
    recv_counts = rc.cpu().numpy()
    rec = hits.dtype.itemsize
    sbuf = torch.from_numpy(send.view(np.uint8).copy()).to(device)
    rbuf = torch.empty(int(recv_counts.sum()) * rec, dtype=torch.uint8, device=device)
    dist.all_to_all_single(rbuf, sbuf, [int(x) * rec for x in recv_counts], [int(x) * rec for x in send_counts])
    got = rbuf.cpu().numpy().view(hits.dtype)
    return _sorted(got)


def combine(local_hits: np.ndarray, n_reads: int, mode: int, dist=None, device="cpu") -> np.ndarray:
    """The exchange step: best-stratum MIN (mode 0) then hits to the read owners."""
    h = best_stratum_filter(local_hits, n_reads, dist, device) if mode == 0 else local_hits
    return exchange_to_owners(h, n_reads, dist, device)


def map_ref_sharded(ctx, reads, ref_codes, chrom_begin, rank: int, world_size: int, params=None, mask=None,
                    dist=None, device="cpu", **kw):
    """One rank's part of a reference-sharded map of a whole read batch on the
    device: plan, upload this rank's pieces, map (all mode), keep owned hits,
    exchange. Returns this rank's reads' hits (whole-reference coordinates)."""
    from . import Reference, make_params

    p = params or make_params(**kw)
    shares = plan(chrom_begin, world_size, reads.stride, p.band_width)
    mine = shares[rank]
    if mine:
        codes, cb, m = piece_reference(ref_codes, chrom_begin, mine, mask)
        R = Reference.from_codes(ctx, codes, cb, mask=m)
        q = make_params(q=p.q, group_width=p.group_width, sampled=p.sampled, band_width=p.band_width,
                        pct_identity=p.pct_identity, mode=1, strands=p.strands)
        local, _ = ctx.map(reads, R, q)
        local = own_and_translate(local, mine)
    else:
        from . import HIT_DTYPE
        local = np.zeros(0, HIT_DTYPE)
    return combine(local, reads.n, p.mode, dist, device)

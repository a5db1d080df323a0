"""Read sharding for multi-GPU runs (one process per GPU, torch.distributed).

Reads are the unit of work: a read's hits depend only on the read and the whole
reference, so every rank maps its own contiguous share
of the reads against its own replica of the reference and nothing crosses
ranks on the data path. Three host-side pieces surround the per-rank map:

  * read_blocks   -- which fixed read blocks a rank maps. A read set is a
                     sequence of blocks (one simulated batch each); weak
                     scaling gives every rank its own blocks_per_rank blocks,
                     strong scaling splits a fixed job's blocks over the ranks,
                     so the whole job's reads are the same at every world size;
  * broadcast_reference -- the 2-bit reference is copied to the device once
                     (rank 0) and broadcast over NVLink (NCCL), instead of G
                     host-to-device copies of the same bytes;
  * HostGather    -- the end-of-run hit gather: all-gather of the per-rank
                     hit counts, prefix offsets, and every rank's records
                     copied into ONE shared host buffer at its offset
                     (POSIX shared memory), where rank 0 reads the whole job's
                     hits. Every GPU keeps its own PCIe link for its D2H; the
                     collective carries only the counts.

The collective layer also carries the barrier and the max-over-ranks timing.
"""
from __future__ import annotations

import os

import numpy as np


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of n reads for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world_size)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def read_blocks(rank: int, world_size: int, blocks_per_rank: int = 1, total_blocks: int | None = None) -> list[int]:
    """Block ids mapped by `rank`: weak scaling (total_blocks None) gives every
    rank blocks [rank*bpr, (rank+1)*bpr); strong scaling splits the job's
    total_blocks contiguously over the ranks."""
    if total_blocks is None:
        return list(range(rank * blocks_per_rank, (rank + 1) * blocks_per_rank))
    b, e = shard_range(total_blocks, rank, world_size)
    return list(range(b, e))


def max_over_ranks(values, dist=None, device="cpu"):
    """Element-wise max of a list of floats over all ranks (identity without dist)."""
    if dist is None or not dist.is_initialized():
        return list(values)
    import torch

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values, dist=None, device="cpu"):
    if dist is None or not dist.is_initialized():
        return list(values)
    import torch

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def weak_scaling_value(units_per_rank: int, steps: int, world_size: int, max_ms: float) -> float:
    """Whole-job throughput: every rank's units over the slowest rank's time."""
    return units_per_rank * steps * world_size / (max_ms / 1e3)


def broadcast_reference(words: np.ndarray | None, n_words: int, dist=None, device="cpu"):
    """The 2-bit reference words as a tensor on `device` on every rank: rank 0
    copies its host words in once, the process group broadcasts them (NCCL
    over NVLink for CUDA devices; gloo broadcasts host tensors, which are then
    copied to the device). Returns (tensor, seconds on this rank)."""
    import time

    import torch

    t0 = time.perf_counter()
    rank = dist.get_rank() if dist is not None and dist.is_initialized() else 0
    nccl = dist is not None and dist.is_initialized() and dist.get_backend() == "nccl"
    on = device if (nccl or dist is None or not dist.is_initialized()) else "cpu"
    if rank == 0:
        t = torch.from_numpy(np.ascontiguousarray(words[:n_words]).view(np.int64)).to(on)
    else:
        t = torch.empty(n_words, dtype=torch.int64, device=on)
    if dist is not None and dist.is_initialized():
        dist.broadcast(t, src=0)
    if str(on) != str(device):
        t = t.to(device)
    if str(device).startswith("cuda"):
        torch.cuda.synchronize(device)
    return t, time.perf_counter() - t0


class HostGather:
    """End-of-run gather of every rank's hit records into one shared host
    buffer at prefix offsets. Collective: every rank calls gather() with its
    records (a numpy structured array); rank 0 gets the whole job's records
    back (others get None). Counts travel through the process group
    (all_gather on `device`); the records through POSIX shared memory."""

    def __init__(self, dist=None, device="cpu", tag: str = "qgm"):
        self.dist, self.device, self.tag = dist, device, tag
        self.last = {}

    def _ranks(self):
        if self.dist is None or not self.dist.is_initialized():
            return 0, 1
        return self.dist.get_rank(), self.dist.get_world_size()

    def gather(self, parts, dtype=None):
        """parts: this rank's records (an array or a list of arrays, laid out
        consecutively). Returns the whole job's records on rank 0 (rank order,
        then part order), None elsewhere; self.last["segments"] = the record
        count of every (rank, part) segment."""
        import time

        import torch

        t0 = time.perf_counter()
        parts = [parts] if isinstance(parts, np.ndarray) else list(parts)
        dtype = dtype or parts[0].dtype
        sizes = [int(p.size) for p in parts]
        rank, G = self._ranks()
        if G == 1:
            self.last = {"method": "single rank (no gather)", "counts": [sum(sizes)], "segments": sizes,
                         "seconds": time.perf_counter() - t0}
            return np.concatenate(parts) if parts else np.zeros(0, dtype)
        dist = self.dist
        # record counts of every part of every rank (ranks may hold different
        # numbers of parts: padded to the largest with -1)
        npart = torch.tensor([len(sizes)], dtype=torch.int64, device=self.device)
        alln = [torch.empty_like(npart) for _ in range(G)]
        dist.all_gather(alln, npart)
        maxp = max(int(x.item()) for x in alln)
        cnt = torch.tensor(sizes + [-1] * (maxp - len(sizes)), dtype=torch.int64, device=self.device)
        allc = [torch.empty_like(cnt) for _ in range(G)]
        dist.all_gather(allc, cnt)
        segs = [int(x) for c in allc for x in c.tolist() if x >= 0]
        counts = [int(c.clamp(min=0).sum().item()) for c in allc]
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        rec = np.dtype(dtype).itemsize
        from multiprocessing import shared_memory

        nbytes = max(int(offs[-1]) * rec, 1)
        # POSIX shared memory (/dev/shm) when it has room for the job's
        # records, else a file-backed mapping under the temp directory (a
        # container's /dev/shm may be a few tens of MB)
        name = [None]
        if rank == 0:
            import shutil
            import tempfile
            try:
                room = shutil.disk_usage("/dev/shm").free
            except OSError:
                room = 0
            if room > 2 * nbytes and not os.environ.get("QGM_GATHER_FILE"):  # (test knob: force the file)
                shm = shared_memory.SharedMemory(create=True, size=nbytes)
                name = [("shm", shm.name)]
            else:
                fd, path = tempfile.mkstemp(prefix=self.tag + "_gather_")
                os.ftruncate(fd, nbytes)
                os.close(fd)
                name = [("file", path)]
        dist.broadcast_object_list(name, src=0)
        kind, where = name[0]
        if kind == "file":
            shm = _FileSegment(where, nbytes, owner=rank == 0)
        elif rank != 0:
            shm = shared_memory.SharedMemory(name=where)
        try:
            buf = np.ndarray((int(offs[-1]),), dtype=dtype, buffer=shm.buf)
            at = int(offs[rank])
            for p in parts:
                buf[at:at + p.size] = p
                at += p.size
            dist.barrier()
            out = buf.copy() if rank == 0 else None
            del buf
            dist.barrier()  # every rank is done with the segment before it goes away
        finally:
            shm.close()
            if rank == 0:
                shm.unlink()
        self.last = {"method": "all_gather(counts) + records into one shared host buffer at prefix offsets "
                               f"({'POSIX shared memory' if kind == 'shm' else 'file mapping'})",
                     "counts": counts, "segments": segs, "bytes": int(offs[-1]) * rec,
                     "seconds": time.perf_counter() - t0}
        return out


class _FileSegment:
    """A file mapping with the SharedMemory interface HostGather uses."""

    def __init__(self, path, nbytes, owner):
        import mmap
        self.path, self.owner = path, owner
        self._f = open(path, "r+b")
        self._m = mmap.mmap(self._f.fileno(), nbytes)
        self.buf = memoryview(self._m)

    def close(self):
        self.buf.release()
        self._m.close()
        self._f.close()

    def unlink(self):
        if self.owner:
            os.unlink(self.path)


def hits_digest(hits: np.ndarray) -> str:
    """sha256 (16 hex) of a hit set in canonical order: (read, chrom, ref_start,
    strand, edits) of every record, sorted -- the parity fingerprint."""
    import hashlib

    if hits.size == 0:
        return hashlib.sha256(b"").hexdigest()[:16]
    cols = [np.asarray(hits[c], dtype=np.int64) for c in ("read_id", "chrom", "ref_start", "strand", "edits")]
    order = np.lexsort(cols[::-1])
    m = np.stack([c[order] for c in cols], axis=1)
    return hashlib.sha256(np.ascontiguousarray(m).tobytes()).hexdigest()[:16]

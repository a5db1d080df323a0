"""World-size-2 gloo tests (CPU) of the multi-GPU plumbing bench.py uses
(paper_1403_1706_b200/sharding.py): read blocks per rank (weak and strong
scaling), the reference broadcast, max-over-ranks timing, and the end-of-run
HostGather of every rank's hits into one shared host buffer. Each rank maps
its blocks with the CPU oracle (the stand-in for its GPU); the gathered hits
must equal the single-process result over the same reads, and the parity
digest must not depend on the world size."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from qgm_testutil import ROOT

L, BLOCK, N_BLOCKS = 200_000, 500, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    import paper_1403_1706_b200 as qgm
    ref = qgm.random_reference(3, L)
    cb = np.array([0, 120_000, L], np.uint64)
    return qgm, ref, cb


def _block(qgm, ref, cb, b):
    codes, lengths, *_ = qgm.simulate_reads(1000 + b, ref, cb, BLOCK, 100, 0.03)
    return codes, lengths


def _worker(rank, world_size, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle.pyoracle import Oracle
    from paper_1403_1706_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    qgm, ref, cb = _data()
    # the reference: rank 0's words broadcast to every rank
    words = qgm.pack_codes(ref) if rank == 0 else None
    t, _ = sharding.broadcast_reference(words, (L + 31) // 32 + 1, dist, "cpu")
    np.save(os.path.join(out_dir, f"ref_{rank}.npy"), t.numpy())
    # strong scaling: the job's N_BLOCKS blocks split over the ranks
    blocks = sharding.read_blocks(rank, world_size, total_blocks=N_BLOCKS)
    parts = []
    for b in blocks:
        codes, lengths = _block(qgm, ref, cb, b)
        hits, _ = Oracle().map(ref, cb, codes, 100, lengths, q=12, mode=1, threads=2)
        parts.append(hits)
    g = sharding.HostGather(dist, "cpu")
    got = g.gather(parts, qgm.HIT_DTYPE)
    mx = sharding.max_over_ranks([float(10 + rank)], dist)
    if rank == 0:
        segs = [b for r in range(world_size) for b in sharding.read_blocks(r, world_size, total_blocks=N_BLOCKS)]
        got["read_id"] += np.repeat(np.array(segs, np.uint64) * BLOCK, g.last["segments"]).astype(np.uint32)
        np.save(os.path.join(out_dir, "gathered.npy"), got)
        np.save(os.path.join(out_dir, "max.npy"), np.array(mx))
        with open(os.path.join(out_dir, "method.txt"), "w") as f:
            f.write(g.last["method"])
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_reads_once():
    from paper_1403_1706_b200 import sharding
    for n in (0, 1, 7, 1000, 1_000_003):
        for w in (1, 2, 3, 8):
            spans = [sharding.shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_read_blocks_weak_and_strong():
    from paper_1403_1706_b200 import sharding
    assert sharding.read_blocks(2, 4, blocks_per_rank=3) == [6, 7, 8]
    for G in (1, 2, 4, 8):
        allb = [b for r in range(G) for b in sharding.read_blocks(r, G, total_blocks=8)]
        assert allb == list(range(8))  # the same job at every world size


def test_weak_scaling_value():
    from paper_1403_1706_b200 import sharding
    assert sharding.weak_scaling_value(1_000_000, 5, 4, 2000.0) == pytest.approx(1e7)


def test_hits_digest_is_order_free():
    import paper_1403_1706_b200 as qgm
    from paper_1403_1706_b200 import sharding
    h = np.zeros(5, qgm.HIT_DTYPE)
    h["read_id"] = [3, 1, 2, 1, 0]
    h["ref_start"] = [9, 8, 7, 6, 5]
    assert sharding.hits_digest(h) == sharding.hits_digest(h[::-1].copy())
    h2 = h.copy()
    h2["edits"][0] = 1
    assert sharding.hits_digest(h) != sharding.hits_digest(h2)


@pytest.mark.parametrize("world_size,via_file", [(2, False), (3, False), (2, True)])
def test_gloo_gather_of_sharded_maps_equals_single_process(tmp_path, oracle, monkeypatch, world_size, via_file):
    from paper_1403_1706_b200 import sharding
    if via_file:  # the file-backed segment used when /dev/shm is too small
        monkeypatch.setenv("QGM_GATHER_FILE", "1")
    port = _free_port()
    mp.start_processes(_worker, args=(world_size, port, str(tmp_path)), nprocs=world_size, join=True,
                       start_method="spawn")
    qgm, ref, cb = _data()
    words = qgm.pack_codes(ref)
    for r in range(world_size):
        assert np.array_equal(np.load(tmp_path / f"ref_{r}.npy").view(np.uint64), words[: (L + 31) // 32 + 1])
    got = np.load(tmp_path / "gathered.npy")
    codes = np.concatenate([_block(qgm, ref, cb, b)[0] for b in range(N_BLOCKS)])
    lengths = np.concatenate([_block(qgm, ref, cb, b)[1] for b in range(N_BLOCKS)])
    whole, _ = oracle.map(ref, cb, codes, 100, lengths, q=12, mode=1, threads=2)
    assert sharding.hits_digest(got) == sharding.hits_digest(whole)
    cols = ("read_id", "chrom", "ref_start", "edits", "strand")
    assert all(np.array_equal(got[c], whole[c]) for c in cols)
    assert float(np.load(tmp_path / "max.npy")[0]) == 10.0 + world_size - 1
    method = (tmp_path / "method.txt").read_text()
    assert ("file mapping" in method) == via_file, method

"""World-size-2 gloo tests (CPU) of the multi-GPU plumbing used by bench.py:
read sharding, max-over-ranks timing and hit-count aggregation. Each rank maps
its shard with the CPU oracle (the stand-in for its GPU) and the union of the
per-rank hits must equal the single-process result: sharding reads changes
nothing but read ids."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from qgm_testutil import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world_size, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle.pyoracle import Oracle
    from paper_1403_1706_b200 import sharding
    import paper_1403_1706_b200 as qgm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    L, N = 200_000, 1_500
    ref = qgm.random_reference(3, L)
    cb = np.array([0, 120_000, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(4, ref, cb, N, 100, 0.03)
    b, e = sharding.shard_range(N, rank, world_size)
    hits, st = Oracle().map(ref, cb, codes[b * 100:e * 100], 100, lengths[b:e], q=12, mode=1, threads=2)
    hits["read_id"] += b
    ms = [float(10 + rank)]
    mx = sharding.max_over_ranks(ms, dist)
    tot = sharding.sum_over_ranks([hits.size], dist)
    np.save(os.path.join(out_dir, f"hits_{rank}.npy"), hits)
    np.save(os.path.join(out_dir, f"red_{rank}.npy"), np.array([mx[0], tot[0]]))
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


def test_weak_scaling_value():
    from paper_1403_1706_b200 import sharding
    assert sharding.weak_scaling_value(1_000_000, 5, 4, 2000.0) == pytest.approx(1e7)


def test_two_rank_gloo_sharded_map_equals_single_process(tmp_path, oracle):
    import paper_1403_1706_b200 as qgm
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"hits_{r}.npy") for r in range(2)]
    red = [np.load(tmp_path / f"red_{r}.npy") for r in range(2)]
    merged = np.concatenate(parts)
    L, N = 200_000, 1_500
    ref = qgm.random_reference(3, L)
    cb = np.array([0, 120_000, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(4, ref, cb, N, 100, 0.03)
    whole, _ = oracle.map(ref, cb, codes, 100, lengths, q=12, mode=1, threads=2)
    cols = ("read_id", "chrom", "ref_start", "edits", "strand")
    assert all(np.array_equal(merged[c], whole[c]) for c in cols)
    assert all(r[0] == 11.0 for r in red)          # max over ranks
    assert all(r[1] == merged.size for r in red)   # hit counts summed

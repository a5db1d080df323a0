"""Reference-sharded mapping (paper_1403_1706_b200/refshard.py, SURVEY 8(f)
row 2) on the CPU: the share plan, and world-size 2 and 3 gloo runs in which
each rank maps the whole read batch against its pieces with the CPU oracle
(the stand-in for its GPU), keeps the hits it owns, and the exchange step
(all-reduce MIN for best-stratum, all-to-all to the read owners) must
reproduce the single-process oracle result exactly -- chromosome cuts,
reads near cuts and chromosome ends, both modes."""
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


def _data():
    import paper_1403_1706_b200 as qgm
    L = 150_000
    ref = qgm.random_reference(13, L)
    # a repeat copied across a future cut so hits straddle shares
    ref[70_000:70_400] = ref[10_000:10_400]
    cb = np.array([0, 90_000, 90_500, L], np.uint64)
    codes, lengths, *_ = qgm.simulate_reads(14, ref, cb, 1200, 100, 0.04)
    return ref, cb, codes, lengths


def test_plan_partitions_every_chromosome():
    from paper_1403_1706_b200 import refshard
    cb = np.array([0, 90_000, 90_500, 150_000], np.uint64)
    for G in (1, 2, 3, 5, 8):
        shares = refshard.plan(cb, G, 100, 32)
        owned = {c: [] for c in range(3)}
        for pieces in shares:
            for p in pieces:
                owned[p.chrom].append((p.own_begin, p.own_end))
                assert p.begin == max(0, p.own_begin - 64)
                assert p.end == min(int(cb[p.chrom + 1] - cb[p.chrom]), p.own_end + 164)
        for c, spans in owned.items():
            spans.sort()
            assert spans[0][0] == 0 and spans[-1][1] == int(cb[c + 1] - cb[c])
            assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
        sizes = [sum(p.own_end - p.own_begin for p in s) for s in shares]
        assert max(sizes) - min(sizes) <= 1


def _worker(rank, world_size, port, out_dir, mode):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle.pyoracle import Oracle
    from paper_1403_1706_b200 import refshard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    ref, cb, codes, lengths = _data()
    mine = refshard.plan(cb, world_size, 100, 32)[rank]
    pc, pcb, _ = refshard.piece_reference(ref, cb, mine)
    local, _ = Oracle().map(pc, pcb, codes, 100, lengths, q=12, mode=1, threads=2)
    local = refshard.own_and_translate(local, mine)
    got = refshard.combine(local, lengths.size, mode, dist)
    np.save(os.path.join(out_dir, f"hits_{rank}.npy"), got)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world_size,mode", [(2, 0), (2, 1), (3, 0), (3, 1)])
def test_reference_sharded_map_equals_single_process(tmp_path, world_size, mode):
    from oracle.pyoracle import Oracle
    from paper_1403_1706_b200 import sharding
    mp.spawn(_worker, args=(world_size, _free_port(), str(tmp_path), mode), nprocs=world_size, join=True)
    ref, cb, codes, lengths = _data()
    want, _ = Oracle().map(ref, cb, codes, 100, lengths, q=12, mode=mode, threads=4)
    parts = [np.load(tmp_path / f"hits_{r}.npy") for r in range(world_size)]
    for r, h in enumerate(parts):  # each rank holds exactly its own reads
        b, e = sharding.shard_range(lengths.size, r, world_size)
        assert np.all((h["read_id"] >= b) & (h["read_id"] < e))
    got = np.concatenate(parts)
    assert got.size == want.size and got.size > 1000
    assert np.array_equal(got, want)


def test_plan_edge_cases_tiny_references_and_empty_chromosomes():
    from paper_1403_1706_b200 import refshard
    # more ranks than bases, and an empty chromosome in the middle
    cb = np.array([0, 3, 3, 5], np.uint64)
    shares = refshard.plan(cb, 8, 100, 32)
    owned = sorted((p.chrom, p.own_begin, p.own_end) for s in shares for p in s)
    assert sum(e - b for _, b, e in owned) == 5
    assert all(c != 1 for c, _, _ in owned)  # the empty chromosome owns nothing
    assert sum(1 for s in shares if not s) >= 3
    # piece references carry the mask slice
    ref = np.arange(5, dtype=np.uint8) % 4
    mask = np.array([0, 1, 0, 1, 1], np.uint8)
    for s in shares:
        codes, pcb, m = refshard.piece_reference(ref, cb, s, mask)
        assert codes.size == int(pcb[-1]) and (m is None or m.size == codes.size)
    # own_and_translate on an empty share keeps nothing
    import paper_1403_1706_b200 as qgm
    h = np.zeros(3, qgm.HIT_DTYPE)
    assert refshard.own_and_translate(h, []).size == 0

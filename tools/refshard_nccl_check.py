"""Reference-sharded mapping over NCCL (torchrun, one rank per GPU): every
rank maps the whole batch against its pieces on its GPU and the exchange runs
on CUDA tensors; rank 0 compares the union with a single-GPU map of the whole
reference. Usage: torchrun --nproc-per-node N tools/refshard_nccl_check.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_1706_b200 as qgm  # noqa: E402
from paper_1403_1706_b200 import refshard, sharding  # noqa: E402

rank, world, local = sharding.world()
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = qgm.Context(local)
L = 2_000_000
ref = qgm.random_reference(5, L)
cb = np.array([0, 700_000, 700_500, L], np.uint64)
codes, lengths, *_ = qgm.simulate_reads(6, ref, cb, 20_000, 100, 0.03)
reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
for mode in (0, 1):
    got = refshard.map_ref_sharded(ctx, reads, ref, cb, rank, world, q=14, mode=mode, dist=dist,
                                   device=f"cuda:{local}")
    parts = [None] * world
    dist.all_gather_object(parts, got.tobytes())
    if rank == 0:
        allh = np.concatenate([np.frombuffer(p, dtype=qgm.HIT_DTYPE) for p in parts])
        want, _ = ctx.map(reads, qgm.Reference.from_codes(ctx, ref, cb), q=14, mode=mode)
        ok = allh.size == want.size and np.array_equal(allh, want)
        print(f"refshard over NCCL, world {world}, mode {mode}: {allh.size} hits (whole reference {want.size}), "
              f"identical={ok}", flush=True)
        if not ok:
            raise SystemExit(1)
dist.barrier()
dist.destroy_process_group()

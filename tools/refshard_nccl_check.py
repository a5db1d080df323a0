"""Reference-sharded mapping across ranks (torchrun, one process per rank):
every rank maps the whole batch against its pieces on its GPU, the records
stay on the device, and the exchange (MIN all-reduce + all-to-all) runs on
CUDA tensors over NCCL; rank 0 compares the union with a single-GPU map of the
whole reference. With fewer GPUs than ranks (a 1-GPU box) the ranks share the
device and the exchange runs over gloo on host copies of the records.
Usage: torchrun --nproc-per-node N tools/refshard_nccl_check.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_1706_b200 as qgm  # noqa: E402
from paper_1403_1706_b200 import refshard, sharding  # noqa: E402

rank, world, local = sharding.world()
n_dev = torch.cuda.device_count()
dev = local % n_dev
torch.cuda.set_device(dev)
nccl = world <= n_dev
if nccl:
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
else:
    dist.init_process_group("gloo")
xdev = f"cuda:{dev}" if nccl else "cpu"
ctx = qgm.Context(dev)
L = 2_000_000
ref = qgm.random_reference(5, L)
ref[1_500_000:1_501_000] = ref[300_000:301_000]  # a repeat across a share cut
cb = np.array([0, 700_000, 700_500, L], np.uint64)
codes, lengths, *_ = qgm.simulate_reads(6, ref, cb, 20_000, 100, 0.03)
reads = qgm.Reads.from_codes(ctx, codes, lengths, 100)
for mode in (0, 1):
    got = refshard.map_ref_sharded(ctx, reads, ref, cb, rank, world, q=14, mode=mode, dist=dist, device=xdev)
    parts = [None] * world
    dist.all_gather_object(parts, refshard.from_records(got).tobytes())
    if rank == 0:
        allh = np.concatenate([np.frombuffer(p, dtype=qgm.HIT_DTYPE) for p in parts])
        want, _ = ctx.map(reads, qgm.Reference.from_codes(ctx, ref, cb), q=14, mode=mode)
        ok = allh.size == want.size and np.array_equal(allh, want)
        print(f"refshard over {'NCCL' if nccl else 'gloo'}, world {world}, mode {mode}: {allh.size} hits "
              f"(whole reference {want.size}), identical={ok}", flush=True)
        if not ok:
            raise SystemExit(1)
dist.barrier()
del reads
ctx.close()
dist.destroy_process_group()

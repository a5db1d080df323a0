"""Distribution of the streamed e2e time per batch for K = 5 (the bench
default) and K = 10, with the bench's NUMA binding."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1403_1706_b200 as qgm
import bench
print("numa cores", bench.bind_to_gpu_numa(0))
cfg = bench.CONFIGS["C2"]
ref, cb, codes, lengths = bench.make_inputs(qgm, cfg, 0)
stream = torch.cuda.Stream(0)
ctx = qgm.Context(0, stream=stream.cuda_stream)
R = qgm.Reference.from_codes(ctx, ref, cb); R.prepare(16)
h_dense = torch.from_numpy(qgm.pack_codes(codes).view(np.int64)).pin_memory()
cap = 1_100_000
h_hits = torch.empty(cap * 16, dtype=torch.uint8).pin_memory()
params = qgm.make_params(q=16, mode=1)
def run(K):
    arr = (qgm.Batch * K)()
    for i in range(K):
        arr[i] = qgm.Batch(h_dense.data_ptr(), None, len(lengths), 100, h_hits.data_ptr(), cap, 0, qgm.MapStats(), 1, 0)
    ctx._check(ctx.lib.qgm_map_host_batches(ctx.h, arr, K, R.h, C.byref(params)))
run(5)
for K in (5, 10, 5):
    ts = []
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(stream); run(K); e1.record(stream); e1.synchronize()
        ts.append(round(e0.elapsed_time(e1) / K, 3))
    print("K", K, ts)

import sys, time, json, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1403_1706_b200 as qgm
import bench
cfg = bench.CONFIGS["C2"]
ref, cb, codes, lengths = bench.make_inputs(qgm, cfg, 0)
stream = torch.cuda.Stream(0)
ctx = qgm.Context(0, stream=stream.cuda_stream)
R = qgm.Reference.from_codes(ctx, ref, cb); R.prepare(16)
words = qgm.pack_read_codes(codes, 100)
h_words = torch.from_numpy(words.view(np.int64)).pin_memory()
h_dense = torch.from_numpy(qgm.pack_codes(codes).view(np.int64)).pin_memory()
DENSE = len(sys.argv) > 1 and sys.argv[1] == "dense"
h_len = torch.from_numpy(lengths.view(np.int32)).pin_memory()
cap = 4_000_000
h_hits = torch.empty(cap * 16, dtype=torch.uint8).pin_memory()
params = qgm.make_params(q=16, mode=1)
lib = ctx.lib
def run(K):
    arr = (qgm.Batch * K)()
    for i in range(K):
        if DENSE:
            arr[i] = qgm.Batch(h_dense.data_ptr(), None, len(lengths), 100, h_hits.data_ptr(), cap, 0, qgm.MapStats(), 1, 0)
        else:
            arr[i] = qgm.Batch(h_words.data_ptr(), h_len.data_ptr(), len(lengths), 100, h_hits.data_ptr(), cap, 0, qgm.MapStats(), 0, 0)
    ctx._check(lib.qgm_map_host_batches(ctx.h, arr, K, R.h, C.byref(params)))
run(3)
for K in (1, 2, 5, 10):
    torch.cuda.synchronize(); t0 = time.perf_counter(); run(K); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print("K", K, "ms/batch", round(t / K * 1e3, 3))
ctx.profile(True); ctx.stage_times(reset=True); ctx.kernel_times(reset=True)
run(5)
print("stages", {k: round(v / 5, 3) for k, v in ctx.stage_times(reset=True, host=True).items() if v})
print("kernels", {k: round(v[0] / v[1], 3) for k, v in ctx.kernel_times(reset=True).items()})
ctx.profile(False)
# host-side timing of a pure compute loop for reference
rd = qgm.Reads(ctx, words, lengths, 100)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): ctx.map(rd, R, q=16, mode=1)
torch.cuda.synchronize(); print("map only ms", round((time.perf_counter() - t0) / 5 * 1e3, 3))

"""Does a preceding device-resident pass (as in bench.py) change the streamed
e2e time? Runs e2e, then device passes, then e2e again."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1403_1706_b200 as qgm
import bench
bench.bind_to_gpu_numa(0)
cfg = bench.CONFIGS["C2"]
ref, cb, codes, lengths = bench.make_inputs(qgm, cfg, 0)
stream = torch.cuda.Stream(0)
ctx = qgm.Context(0, stream=stream.cuda_stream)
R = qgm.Reference.from_codes(ctx, ref, cb); R.prepare(16)
h_dense = torch.from_numpy(qgm.pack_codes(codes).view(np.int64)).pin_memory()
cap = len(lengths) * 4
h_hits = torch.empty(cap * 16, dtype=torch.uint8).pin_memory()
params = qgm.make_params(q=16, mode=1)
words = qgm.pack_read_codes(codes, 100)
d_words = torch.from_numpy(words.view(np.int64)).to("cuda:0")
d_len = torch.from_numpy(lengths.view(np.int32)).to("cuda:0")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
lib = ctx.lib
def run(K):
    arr = (qgm.Batch * K)()
    for i in range(K):
        arr[i] = qgm.Batch(h_dense.data_ptr(), None, len(lengths), 100, h_hits.data_ptr(), cap, 0, qgm.MapStats(), 1, 0)
    ctx._check(lib.qgm_map_host_batches(ctx.h, arr, K, R.h, C.byref(params)))
def dev():
    rd = C.c_void_p()
    ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(d_words.data_ptr()), C.c_void_p(d_len.data_ptr()), len(lengths), 100, C.byref(rd)))
    h = C.c_void_p()
    ctx._check(lib.qgm_map(ctx.h, rd, R.h, C.byref(params), C.byref(h)))
    lib.qgm_hits_destroy(h); lib.qgm_reads_destroy(rd)
def t_e2e(tag):
    run(5)
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(stream); run(5); e1.record(stream); e1.synchronize()
        ts.append(round(e0.elapsed_time(e1) / 5, 3))
    print(tag, ts, flush=True)
t_e2e("fresh")
for _ in range(8):
    with torch.cuda.stream(stream): flush.fill_(1)
    dev()
torch.cuda.synchronize()
t_e2e("after device passes")
ctx.profile(True); dev(); ctx.profile(False)
t_e2e("after a profiled pass")

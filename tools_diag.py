import sys, time, os, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1403_1706_b200 as qgm
L, N = 100_000_000, 1_000_000
ref = qgm.random_reference(7, L); cb = np.array([0, L], np.uint64)
codes, lengths, *_ = qgm.simulate_reads(1000, ref, cb, N, 100, 0.03)
words = qgm.pack_read_codes(codes, 100)
for variant in ("own_stream", "torch_stream"):
    if variant == "torch_stream":
        stream = torch.cuda.Stream(0); ctx = qgm.Context(0, stream=stream.cuda_stream)
    else:
        ctx = qgm.Context(0)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    t0 = time.perf_counter(); R.prepare(16); print(variant, "prepare", round(time.perf_counter() - t0, 3), flush=True)
    d_words = torch.from_numpy(words.view(np.int64)).cuda(); d_len = torch.from_numpy(lengths.view(np.int32)).cuda()
    params = qgm.make_params(q=16, mode=1)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    lib = ctx.lib
    for it in range(6):
        if it >= 3: flush.fill_(1); torch.cuda.synchronize()
        t0 = time.perf_counter()
        rd = C.c_void_p()
        ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(d_words.data_ptr()), C.c_void_p(d_len.data_ptr()), N, 100, C.byref(rd)))
        t1 = time.perf_counter()
        h = C.c_void_p()
        ctx._check(lib.qgm_map(ctx.h, rd, R.h, C.byref(params), C.byref(h)))
        t2 = time.perf_counter()
        lib.qgm_hits_destroy(h); lib.qgm_reads_destroy(rd); ctx.synchronize()
        print(variant, it, "reads", round((t1-t0)*1e3, 2), "map", round((t2-t1)*1e3, 2), "flush" if it >= 3 else "", flush=True)
    del R
    ctx.close()

"""Host-side cost of one small batch (C1 shape: 10k x 100 bp, 1 Mbp) through
the C ABI: wall time per call of qgm_reads_from_device, qgm_map and the
handle releases, against the GPU time of the map (CUDA events), so that a
launch- or host-bound configuration shows up as wall >> GPU."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1403_1706_b200 as qgm  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
ref, cb = bench.make_reference(qgm, cfg)
codes, lengths = bench.make_block(qgm, cfg, ref, cb, 0)
stream = torch.cuda.Stream()
ctx = qgm.Context(0, stream=stream.cuda_stream)
R = qgm.Reference.from_codes(ctx, ref, cb)
R.prepare(cfg["q"])
lib = ctx.lib
words = torch.from_numpy(qgm.pack_read_codes(codes, cfg["rlen"]).view(np.int64)).cuda()
lens = torch.from_numpy(lengths.view(np.int32)).cuda()
p = qgm.make_params(q=cfg["q"], mode=cfg["mode"], band_width=cfg["band"], pct_identity=cfg["pct"])
T = {"reads": 0.0, "map": 0.0, "release": 0.0}
N = 200
gpu = []
for it in range(N + 20):
    t0 = time.perf_counter()
    rd = C.c_void_p()
    ctx._check(lib.qgm_reads_from_device(ctx.h, C.c_void_p(words.data_ptr()), C.c_void_p(lens.data_ptr()),
                                         lengths.size, cfg["rlen"], C.byref(rd)))
    t1 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h = C.c_void_p()
    ctx._check(lib.qgm_map(ctx.h, rd, R.h, C.byref(p), C.byref(h)))
    e1.record(stream)
    t2 = time.perf_counter()
    lib.qgm_hits_destroy(h)
    lib.qgm_reads_destroy(rd)
    t3 = time.perf_counter()
    e1.synchronize()
    if it >= 20:
        T["reads"] += t1 - t0
        T["map"] += t2 - t1
        T["release"] += t3 - t2
        gpu.append(e0.elapsed_time(e1))
print({k: round(v / N * 1e6, 1) for k, v in T.items()}, "us per call (host wall);",
      "map GPU interval", round(float(np.median(gpu)) * 1e3, 1), "us")

"""Debug probe (variant build with -DQGM_VAL_HIST): where validation abandons
candidates (row / 16 buckets, last = ran to the end)."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_1403_1706_b200 as qgm
import bench
for name in sys.argv[1:] or ["C2"]:
    cfg = bench.CONFIGS[name]
    ref, cb, codes, lengths = bench.make_inputs(qgm, cfg, 0)
    ctx = qgm.Context(0)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    rd = qgm.Reads.from_codes(ctx, codes, lengths, cfg[3])
    lib = ctx.lib
    h = (C.c_ulonglong * 16)()
    lib.qgm_debug_validate_hist(h)
    before = np.array(h[:], np.int64)
    hits, st = ctx.map(rd, R, q=cfg[5], mode=cfg[6])
    lib.qgm_debug_validate_hist(h)
    d = np.array(h[:], np.int64) - before
    print(name, st, "exit-row histogram (x16):", d.tolist())

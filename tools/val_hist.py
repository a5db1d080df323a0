"""Abandon-row histogram of the validation (rows / 16 at which a candidate's
lower bound passed k_max; the last bin = ran every row), one map of a bench
config's first batch without the phase split. Needs a library built with
-DQGM_VAL_HIST:
    bash tools/build_variant.sh vhist validate.cu -DQGM_VAL_HIST
    QGM_LIB=build/var_vhist.so QGM_VAL_SPLIT=1008 python tools/val_hist.py C2"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(config):
    import bench
    import paper_1403_1706_b200 as qgm

    cfg = bench.CONFIGS[config]
    ref, cb = bench.make_reference(qgm, cfg)
    codes, lengths = bench.make_block(qgm, cfg, ref, cb, 0)
    ctx = qgm.Context(0)
    R = qgm.Reference.from_codes(ctx, ref, cb)
    if cfg["mask_threshold"]:
        R.mask_repeats(cfg["q"], cfg["mask_threshold"])
    R.prepare(cfg["q"])
    reads = qgm.Reads.from_codes(ctx, codes, lengths, cfg["rlen"])
    p = qgm.make_params(q=cfg["q"], mode=cfg["mode"], band_width=cfg["band"], pct_identity=cfg["pct"])
    lib = C.CDLL(qgm.LIB_PATH)
    h0 = (C.c_ulonglong * 16)()
    lib.qgm_debug_validate_hist(h0)
    _, st = ctx.map(reads, R, p)
    h1 = (C.c_ulonglong * 16)()
    lib.qgm_debug_validate_hist(h1)
    hist = [int(b - a) for a, b in zip(h1, h0)] if False else [int(b) - int(a) for a, b in zip(h0, h1)]
    tot = sum(hist) or 1
    mean_rows = sum(16 * (i + 1) * v for i, v in enumerate(hist[:15])) / tot
    print(json.dumps({"config": config, "hist_rows_div16": hist, "unique": st.get("unique_candidates"),
                      "mean_abandon_or_end_rows_upper": mean_rows, "ran_to_end": hist[15]}))
    del reads, R
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1])

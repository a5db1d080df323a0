"""ncu evidence per bench config, stamped with the library build it measured.

    # on the GPU box: one map of the config's first batch under ncu (after an
    # unprofiled warm-up map; cudaProfilerStart/Stop bracket the measured one)
    ncu --profile-from-start off --clock-control none --metrics \
        gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
        --csv --log-file gpurun_out/ncu_C2.csv python tools/ncu_capture.py run C2
    # here: fold the CSV into profiles/<round>/ncu_C2.json (read by bench.py)
    python tools/ncu_capture.py parse C2 gpurun_out/ncu_C2.csv profiles/r02

bench.py uses `kernels.<name>.dram_bytes` as roofline.traffic and
`kernels.k_validate.warp_inst` for the validation issue rate only when
`lib_sha` equals the build stamp (sha256 of the CUDA sources and Makefile)
of the library it runs.
"""
import csv
import io
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# ncu kernel name pattern -> bench.py KernelScope name
NAMES = [("k_join", r"k_join"), ("k_part_hist", r"k_part_hist"), ("k_part_scatter", r"k_part_scatter"),
         ("k_refine_scatter", r"k_refine_scatter"), ("k_validate", r"k_validate"),
         ("k_hash_insert", r"k_hash_insert"), ("k_strata_seg", r"k_seg_|k_scatter_reads"),
         ("k_tile_compact", r"k_tile_compact")]


def run(config):
    import ctypes as C

    import numpy as np
    import torch

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
    _, st = ctx.map(reads, R, p)  # warm-up (allocations, reference tables)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    _, st = ctx.map(reads, R, p)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(json.dumps(st))
    del reads, R
    ctx.close()


def parse(config, csv_path, out_dir):
    import paper_1403_1706_b200 as qgm
    text = open(csv_path).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.DictReader(io.StringIO(text)))
    kern = {}
    for r in rows:
        name = r["Kernel Name"]
        for short, pat in NAMES:
            if re.search(pat, name):
                k = kern.setdefault(short, {"dram_bytes": 0.0, "warp_inst": 0.0, "ms": 0.0, "launches": set(),
                                            "ncu_names": set()})
                v = float(r["Metric Value"].replace(",", ""))
                m, unit = r["Metric Name"], r.get("Metric Unit", "")
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
                if m.startswith("dram__bytes"):
                    k["dram_bytes"] += v * scale.get(unit, 1)
                elif m == "smsp__inst_executed.sum":
                    k["warp_inst"] += v
                elif m == "gpu__time_duration.sum":
                    k["ms"] += v * scale.get(unit, 1e-6)
                k["launches"].add(r["ID"])
                k["ncu_names"].add(name.split("(")[0])
                break
    for k in kern.values():
        k["launches"] = len(k["launches"])
        k["ncu_names"] = sorted(k["ncu_names"])
    sha = qgm.build_stamp()
    os.makedirs(out_dir, exist_ok=True)
    out = {"config": config, "lib_sha": sha, "what": "one map of the config's first batch under ncu "
           "(--clock-control none; per-kernel sums over the launches of that map)", "kernels": kern}
    p = os.path.join(out_dir, f"ncu_{config}.json")
    json.dump(out, open(p, "w"), indent=1)
    print(p, json.dumps({k: (round(v["dram_bytes"] / 1e6, 1), round(v["ms"], 4)) for k, v in kern.items()}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        parse(sys.argv[2], sys.argv[3], sys.argv[4])

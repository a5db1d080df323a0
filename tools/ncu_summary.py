"""Summarise an ncu report (--page raw) into a markdown table: per kernel
duration, DRAM bytes, DRAM throughput %, SM throughput %, achieved occupancy,
L2 hit rate. Usage: python tools/ncu_summary.py report.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("lts__t_sector_hit_rate.pct", "L2hit%"), ("launch__registers_per_thread", "regs"),
        ("smsp__inst_executed.sum", "inst")]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    hdr, units, data = rows(rep)
    idx = {k: hdr.index(k) for k, _ in COLS if k in hdr}
    name_i = hdr.index("Kernel Name")
    print("| kernel | " + " | ".join(n for k, n in COLS if k in idx) + " |")
    print("|---" * (1 + len(idx)) + "|")
    for d in data:
        nm = re.sub(r"\(.*", "", d[name_i]).replace("unnamed>::", "").replace("void ", "").strip()
        if pat and not pat.search(nm):
            continue
        vals = []
        for k, n in COLS:
            if k not in idx:
                continue
            v, u = d[idx[k]], units[idx[k]]
            vals.append(f"{v} {u}".strip())
        print(f"| {nm} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()

"""Per-source-line executed instructions (warp level) and average active
threads of one kernel in an ncu report (--import-source, -lineinfo).
Usage: python tools/ncu_inst.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "-c", "1", "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    res, fname, hdr = [], "?", None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].rsplit("/", 1)[-1]
        elif row[0] == "Line No":
            hdr = row
        elif hdr and row[0] not in ("", "Function Name") and len(row) == len(hdr):
            res.append((fname, row))
    ie, th = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
    f = lambda v: float(v) if v not in ("", "-") else 0.0
    tot = sum(f(r[ie]) for _, r in res) or 1
    print(f"total warp instructions {tot:.4g}")
    for fn, r in sorted(res, key=lambda t: -f(t[1][ie]))[:top]:
        i = f(r[ie])
        avg = f(r[th]) / i if i else 0
        print(f"{100 * i / tot:5.1f}% {fn}:{r[0]:<5} thr/inst={avg:4.1f}  {r[1].strip()[:80]}")


if __name__ == "__main__":
    main()

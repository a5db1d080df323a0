"""Per-source-line warp-stall summary of one kernel in an ncu report
(`--print-source cuda,sass`; needs -lineinfo). Usage:
python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
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
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [(i, c[6:]) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
    f = lambda v: float(v) if v not in ("", "-") else 0.0
    tot = sum(f(r[ws]) for _, r in res) or 1
    for fn, r in sorted(res, key=lambda t: -f(t[1][ws]))[:top]:
        st = sorted(((f(r[i]), c) for i, c in cols), reverse=True)[:3]
        st = " ".join(f"{c}={v / tot * 100:.1f}" for v, c in st if v)
        print(f"{f(r[ws]) / tot * 100:5.1f}% {fn}:{r[0]:<4} {r[1].strip()[:70]:70} | {st}")


if __name__ == "__main__":
    main()

"""Per-CUDA-source-line instruction / stall totals of one kernel in an .ncu-rep.

usage: python tools/src_hot.py REP KERNEL_REGEX [TOP] [SORT_COLUMN]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
key = sys.argv[4] if len(sys.argv) > 4 else "Instructions Executed"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name-base", "demangled", "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0] not in ("", "Function Name"):
        rows.append((fname, r))


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


ki = hdr.index(key)
si = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(num(r[ki]) for _, r in rows)
tots = sum(num(r[si]) for _, r in rows)
print(f"{key}: total {tot:.4g}; stall samples {tots:.4g}")
for f, r in sorted(rows, key=lambda t: -num(t[1][ki]))[:top]:
    print(f"{100*num(r[ki])/tot:5.1f}% inst {100*num(r[si])/max(tots,1):5.1f}% stall  {f}:{r[0]:<5} {r[1].strip()[:80]}")

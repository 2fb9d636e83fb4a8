"""Rank SASS instructions of one kernel in an .ncu-rep by a stall column.

usage: python tools/sass_hot.py REP KERNEL_REGEX [COLUMN] [TOP]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
col = sys.argv[3] if len(sys.argv) > 3 else "stall_long_sb"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ci, si, ai = h.index(col), h.index("Source"), h.index("Address")
ii = h.index("Instructions Executed")
def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


body = [r for r in rows[1:] if len(r) == len(h) and num(r[ci]) is not None]
tot = sum(num(r[ci]) for r in body)
idx = {r[ai]: k for k, r in enumerate(body)}
print(f"{col}: total {tot:.0f} samples, {len(body)} instructions")
for r in sorted(body, key=lambda r: -num(r[ci]))[:top]:
    k = idx[r[ai]]
    print(f"{num(r[ci]):8.0f} {100*num(r[ci])/max(tot,1):5.1f}%  {r[ai]}  {r[si][:90]}")

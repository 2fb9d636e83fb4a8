"""Executed-instruction histogram by SASS opcode for one kernel of an .ncu-rep.

usage: python tools/op_hist.py REP KERNEL_REGEX [REP2]   (two reports: side by side)
"""
import collections
import csv
import io
import subprocess
import sys


def hist(rep, kern):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    si, ii, ai = h.index("Source"), h.index("Instructions Executed"), h.index("Address")
    c = collections.Counter()
    seen = set()
    for r in rows[1:]:
        if len(r) != len(h) or r[ai] in seen:
            continue
        seen.add(r[ai])
        try:
            n = float(r[ii].replace(",", ""))
        except ValueError:
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        c[op.split(".")[0]] += n
    return c


a = hist(sys.argv[1], sys.argv[2])
b = hist(sys.argv[3], sys.argv[2]) if len(sys.argv) > 3 else None
keys = sorted(set(a) | set(b or {}), key=lambda k: -(a.get(k, 0) + (b or {}).get(k, 0)))
print(f"{'op':10} {'A (M)':>9} {'B (M)':>9}")
print(f"{'TOTAL':10} {sum(a.values())/1e6:9.1f} {sum((b or {}).values())/1e6:9.1f}")
for k in keys[:30]:
    print(f"{k:10} {a.get(k,0)/1e6:9.1f} {(b or {}).get(k,0)/1e6:9.1f}")

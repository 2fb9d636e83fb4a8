"""Stall samples and executed instructions per SASS opcode (and top stalled
instructions) of one kernel in an ncu source-page CSV export:
    ncu -i REP --page source --csv --print-source sass --kernel-name-base demangled \
        --kernel-name regex:K > k.csv; python tools/sass_ops.py k.csv [TOP]"""
import collections
import csv
import io
import sys

lines = open(sys.argv[1]).read().splitlines()
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
st = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i, l in enumerate(lines) if i > st and l.startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[st:end]))))
h = rows[0]
si, wi, ii = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg, aggi, tot, per = collections.Counter(), collections.Counter(), 0.0, []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    toks = r[si].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    w = float(r[wi] or 0)
    agg[op] += w
    aggi[op] += float(r[ii] or 0)
    tot += w
    per.append((w, r[h.index("Address")], r[si].strip()))
print(f"stall samples {tot:.0f}, instructions {sum(aggi.values())/1e6:.1f}M")
for k, v in agg.most_common(top):
    print(f"  {k:22s} {100 * v / tot:5.1f}% of stalls  {aggi[k] / 1e6:7.2f}M inst")
print("top instructions:")
for w, a, s in sorted(per, reverse=True)[:top]:
    print(f"  {100 * w / tot:5.2f}%  {a[-5:]}  {s[:90]}")

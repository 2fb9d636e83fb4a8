"""Summarise an ncu report (--set full) or an ncu launch-list CSV as markdown.

    python tools/ncu_summary.py report.ncu-rep [title]
    python tools/ncu_summary.py launches.csv [title]
"""
import csv
import collections
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def summarize_report(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = [f"## {title}", "", f"Source: `{path}` (ncu --set full --clock-control none; caches flushed between "
           "replays, so DRAM bytes are cold-cache upper bounds).", ""]
    names = [r[idx["Kernel Name"]].split("(")[0].replace("void ", "") for r in rows[2:]]
    out.append("| metric | " + " | ".join(names) + " |")
    out.append("|---|" + "---|" * len(names))
    for key, label in KEYS:
        if key not in idx:
            continue
        vals = [r[idx[key]] for r in rows[2:]]
        out.append(f"| {label} ({units[idx[key]]}) | " + " | ".join(vals) + " |")
    stall_rows = []
    for r in rows[2:]:
        st = []
        for h in hdr:
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    st.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[idx[h]].replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(v for _, v in st) or 1.0
        stall_rows.append(", ".join(f"{h} {100 * v / tot:.0f}%" for h, v in sorted(st, key=lambda x: -x[1])[:6]))
    out.append("| top stall reasons | " + " | ".join(stall_rows) + " |")
    return "\n".join(out)


def summarize_launches(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    d = collections.defaultdict(list)
    for r in data:
        if r[im] == "gpu__time_duration.sum":
            d[r[ik].split("(")[0].replace("void ", "")].append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = [f"## {title}", "", f"Source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none; "
           "serialised, cold-cache launches: compare shares, not absolutes).", "",
           "| kernel | launches | mean duration (us) | share |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    p = sys.argv[1]
    t = sys.argv[2] if len(sys.argv) > 2 else p
    print(summarize_report(p, t) if p.endswith(".ncu-rep") else summarize_launches(p, t))

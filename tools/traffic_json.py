"""DRAM bytes per launch / per pair of the mode-A passes from an ncu --set full report.

usage: python tools/traffic_json.py REP PAIRS_PER_LAUNCH SOURCE_NOTE > profiles/r2_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep, pairs, note = sys.argv[1], int(sys.argv[2]), sys.argv[3]
OPS = ["smsp__sass_thread_inst_executed_op_%s_pred_on.sum.per_cycle_elapsed" % o for o in ("fadd", "fmul", "ffma")]
PEAK = "sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained"
CLK = "smsp__cycles_elapsed.avg.per_second"
ISSUE = "smsp__issue_active.avg.pct_of_peak_sustained_active"
FMA = "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      ",".join(["dram__bytes_read.sum", "dram__bytes_write.sum", *OPS, PEAK, CLK, ISSUE, FMA])],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
kern = {}
for r in rows[2:]:
    name = r[ki].replace("(anonymous namespace)::", "")
    name = name.split("(")[0].replace("gtb::", "").replace("void ", "")
    b = float(r[ri].replace(",", "")) * scale[units[ri]] + float(r[wi].replace(",", "")) * scale[units[wi]]
    f = lambda k: float(r[h.index(k)].replace(",", ""))
    fadd, fmul, ffma = (f(k) for k in OPS)
    peak = f(PEAK)  # FP32 lanes per cycle, whole GPU
    kern[name] = {"dram_bytes_per_launch": b, "pairs_per_launch": pairs, "dram_bytes_per_pair": b / pairs,
                  "fp32": {"inst_frac_of_peak": (fadd + fmul + ffma) / peak,
                           "tflops": (fadd + fmul + 2 * ffma) * f(CLK) * 1e9 / 1e12,
                           "peak_tflops_at_clock": 2 * peak * f(CLK) * 1e9 / 1e12,
                           "fma_pipe_active_pct": f(FMA), "issue_active_pct": f(ISSUE)}}
print(json.dumps({"source": note, "kernels": kern}, indent=1))

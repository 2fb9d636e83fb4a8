"""DRAM bytes per launch / per pair of the mode-A passes from an ncu --set full report.

usage: python tools/traffic_json.py REP PAIRS_PER_LAUNCH SOURCE_NOTE > profiles/r1_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep, pairs, note = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
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
    kern[name] = {"dram_bytes_per_launch": b, "pairs_per_launch": pairs, "dram_bytes_per_pair": b / pairs}
print(json.dumps({"source": note, "kernels": kern}, indent=1))

"""Copy one profiling round's artefacts from gpurun_out/ into profiles/.

usage: python tools/refresh_profiles.py VERSION
  gpurun_out/bench_VERSION.json          -> profiles/r1_bench_b200.json (last line, pretty)
  gpurun_out/launches_VERSION.csv        -> profiles/r1_launches.csv
  gpurun_out/prof_r1_modeA_VERSION.ncu-rep -> profiles/r1_traffic.json (DRAM bytes, FP32 use)
Prints the ncu summary table and the launch-list table for the markdown summary.
"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
v = sys.argv[1]
go, pr = ROOT / "gpurun_out", ROOT / "profiles"
line = json.loads((go / f"bench_{v}.json").read_text().strip().splitlines()[-1])
(pr / "r1_bench_b200.json").write_text(json.dumps(line, indent=1) + "\n")
shutil.copy(go / f"launches_{v}.csv", pr / "r1_launches.csv")
rep = go / f"prof_r1_modeA_{v}.ncu-rep"
note = (f"profiles/r1_ncu_summary.md {v}: ncu --set full --clock-control none --cache-control none, "
        "tools/prof_mc.py 1024 1024 (--launch-skip 3: the second 1024-pair batch, one launch per pass); "
        "DRAM = dram__bytes_read.sum + dram__bytes_write.sum; fp32 = smsp__sass_thread_inst_executed_op_"
        "{fadd,fmul,ffma}_pred_on rates vs sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained")
out = subprocess.run([sys.executable, str(ROOT / "tools/traffic_json.py"), str(rep), "1024", note],
                     capture_output=True, text=True, check=True).stdout
d = json.loads(out)
d["kernels"] = {k.replace(", 1>", ">").replace(", true>", ">"): x for k, x in d["kernels"].items()}
(pr / "r1_traffic.json").write_text(json.dumps(d, indent=1) + "\n")
for a in (str(rep), str(pr / "r1_launches.csv")):
    t = subprocess.run([sys.executable, str(ROOT / "tools/ncu_summary.py"), a, v], capture_output=True, text=True).stdout
    print(t[t.index("|"):].strip(), "\n")

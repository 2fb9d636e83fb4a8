"""Small fixed workload for ncu: fp32 mode-A batches (warm-up + profiled).
argv: B chunk prec mu_per_sample(0/1/both) fp64_check"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens, SAMPLE_STATS_DTYPE

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 32
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
mus = sys.argv[4] if len(sys.argv) > 4 else "1"
chk = float(sys.argv[5]) if len(sys.argv) > 5 else -1.0
dt = torch.float64 if prec else torch.float32
P, V = inputs.mc_inputs(inputs.CONFIGS["cfg1"], 0, B, device="cuda", torch_dtype=dt)
dg = DeviceGreens(greens_cfg1(), prec)
out = torch.empty_like(P)
st = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for mu in ([0, 1] if mus == "both" else [int(mus)]):
    for _ in range(2):
        dg.mc_batch_device(P.data_ptr(), V.data_ptr(), B, dg.opts(chunk=chunk, mu_per_sample=mu, fp64_check=chk),
                           out.data_ptr(), st.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
print("done")

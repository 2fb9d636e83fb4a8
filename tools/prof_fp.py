"""Small fixed workload for ncu: fp32 mode-B (linear law) batches (warm-up + profiled)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dt = torch.float64 if prec else torch.float32
P, V = inputs.mc_inputs(inputs.CONFIGS["cfg1"], 0, B, device="cuda", torch_dtype=dt)
dg = DeviceGreens(greens_cfg1(), prec)
out = torch.empty_like(P)
it = torch.zeros(B, dtype=torch.int32, device="cuda")
st = torch.zeros(B, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
accel = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lin = dg.fp_opts(leak_frac=0.3, law=0, kirchhoff=0, beta=0.017, tol=1e-4 if accel else 2e-4, max_iters=200, accel=accel)
for _ in range(2):
    dg.fp_batch_device(P.data_ptr(), V.data_ptr(), B, lin, out.data_ptr(), it.data_ptr(), st.data_ptr(), None, None,
                       s.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
dg.fp_batch_device(P.data_ptr(), V.data_ptr(), B, lin, out.data_ptr(), it.data_ptr(), st.data_ptr(), None, None,
                   s.cuda_stream)
e1.record(s)
torch.cuda.synchronize()
print(f"B={B} ms={e0.elapsed_time(e1):.2f} mean_it={it.float().mean().item():.2f} max_it={it.max().item()}")

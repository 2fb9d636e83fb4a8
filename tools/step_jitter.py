"""Per-step device time of the mode-A batch (config 1) over many steps: looks for
sporadic gaps between steps (development helper)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens, SAMPLE_STATS_DTYPE

B = 4096
P, V = inputs.mc_inputs(inputs.CONFIGS["cfg1"], 0, B, device="cuda", torch_dtype=torch.float32)
dg = DeviceGreens(greens_cfg1(), 0)
out = torch.empty_like(P)
st = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
opts = dg.opts(leak_frac=0.3, mu_per_sample=1, with_rand=1)
mode = int(sys.argv[1]) if len(sys.argv) > 1 else -1  # -1: no profiling marks
prof = mode >= 0
t0 = time.time()
while time.time() - t0 < 1.0:
    dg.mc_batch_device(P.data_ptr(), V.data_ptr(), B, opts, out.data_ptr(), st.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
for rep in range(5):
    N = 20
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
    if prof:
        dg.profile_begin(mode)
    torch.cuda.synchronize()
    ev[0].record(s)
    for i in range(N):
        dg.mc_batch_device(P.data_ptr(), V.data_ptr(), B, opts, out.data_ptr(), st.data_ptr(), s.cuda_stream)
        ev[i + 1].record(s)
    torch.cuda.synchronize()
    if prof:
        dg.profile_end()
    d = [ev[i].elapsed_time(ev[i + 1]) for i in range(N)]
    print(f"rep {rep}: mean {sum(d)/N:.3f} ms  min {min(d):.3f}  max {max(d):.3f}  " +
          " ".join(f"{x:.2f}" for x in d), flush=True)

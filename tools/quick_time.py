"""Quick device-resident timing of the mode-A batch (development helper)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens, GreensArrays, SAMPLE_STATS_DTYPE

z = np.load(Path(__file__).resolve().parents[1] / "tests/golden/greens_n256.npz")
f = z["f_sp0"]; n = int(z["n"]); c = n // 2
g = GreensArrays(n=n, pitch=float(z["pitch"]), f_sp0=f, g_sp0=f + (f[c, c] - float(z["kappa_inf"])), phi=float(z["phi"]),
                 kappa_inf=float(z["kappa_inf"]), alpha=float(z["alpha"]), beta=float(z["beta"]), mu=float(z["mu"]), rand_scale=1.0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = inputs.CONFIGS["cfg1"]
t = time.time()
p, v = inputs.mc_inputs(cfg, 0, B, device="cuda")
torch.cuda.synchronize(); print("inputs", time.time() - t, flush=True)
for prec, dt in ((0, torch.float32), (1, torch.float64)):
    dg = DeviceGreens(g, prec)
    pp, vv = p.to(dt), v.to(dt)
    out = torch.empty_like(pp)
    stats = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for chunk in (16, 32, 64, 128):
        o = dg.opts(chunk=chunk)
        for _ in range(2):
            dg.mc_batch_device(pp.data_ptr(), vv.data_ptr(), B, o, out.data_ptr(), stats.data_ptr(), s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        R = 5
        for _ in range(R):
            dg.mc_batch_device(pp.data_ptr(), vv.data_ptr(), B, o, out.data_ptr(), stats.data_ptr(), s.cuda_stream)
        e1.record(s); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        print(f"prec={prec} chunk={chunk} B={B}: {ms:.3f} ms/batch  {B/ms*1e3:.0f} solves/s  "
              f"{6.05e6*B/ms/1e6:.0f} GB/s(model)", flush=True)
    st = np.frombuffer(stats.cpu().numpy().tobytes(), dtype=SAMPLE_STATS_DTYPE)
    print("status nonzero:", int((st['status'] != 0).sum()), "max rise range", st['max_rise'].min(), st['max_rise'].max())

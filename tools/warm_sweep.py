"""Mode-B iterations from T_0 = 0 vs T_0 = the mode-A closed-form map (per-sample mu, no
shift-variant term: the uniform-leakage approximation of the same fixed point)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens

B = 256
P, V = inputs.mc_inputs(inputs.CONFIGS["cfg1"], 0, B, device="cuda", torch_dtype=torch.float64)
p, v = P.cpu().numpy(), V.cpu().numpy()
g = greens_cfg1()
import dataclasses
dg = DeviceGreens(dataclasses.replace(g, alpha=0.0), 1)
ta = dg.mc_batch_host(p, v, dg.opts(leak_frac=0.3, mu_per_sample=1, with_rand=0))[0]
dgb = DeviceGreens(g, 1)
kw = dict(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
ref = dgb.fp_batch_host(p, v, dgb.fp_opts(**kw))
print("closed form vs fixed point: max |dT|", np.abs(ta - ref[0]).max(), "K")
for acc in (0, 3, 5):
    cold = dgb.fp_batch_host(p, v, dgb.fp_opts(accel=acc, **kw))
    warm = dgb.fp_batch_host(p, v, dgb.fp_opts(accel=acc, warm_start=1, **kw), t0=ta)
    print(f"accel={acc}: cold {cold[1].mean():.2f} (max {cold[1].max()}), warm {warm[1].mean():.2f} (max {warm[1].max()}); "
          f"warm vs cold max|dT| {np.abs(warm[0] - ref[0]).max():.2e} K")

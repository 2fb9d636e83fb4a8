"""Mean mode-B iterations on config-1 pairs for plain Picard and Chebyshev start k0."""
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
dg = DeviceGreens(greens_cfg1(), 1)
p, v = P.cpu().numpy(), V.cpu().numpy()
for law, kir, sc in ((0, 0, 1.0), (1, 0, 0.25), (1, 1, 0.15)):
    base = None
    for k0 in (0, 3, 4, 5, 6, 8):
        out, it, st, _, ms = dg.fp_batch_host(p * sc, v, dg.fp_opts(leak_frac=0.3, beta=0.017, law=law, kirchhoff=kir,
                                                                      tol=1e-4, max_iters=200, accel=k0))
        if base is None:
            base = out
        print(f"law={law} kir={kir} k0={k0}: mean iters {it.mean():.2f} max {it.max()} failed {(st != 0).sum()} "
              f"max|dT| vs Picard {np.abs(out - base).max():.2e} K", flush=True)

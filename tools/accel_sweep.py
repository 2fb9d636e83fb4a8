"""Mean mode-B iterations on config-1 pairs for plain Picard (0), Chebyshev from iteration k0 (> 0)
and Anderson(m) on the low cosine modes (-m), fp64 and fp32 (+ fp64 finish) handles."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
P, V = inputs.mc_inputs(inputs.CONFIGS["cfg1"], 0, B, device="cuda", torch_dtype=torch.float64)
p, v = P.cpu().numpy(), V.cpu().numpy()
for prec in (1, 0):
    dg = DeviceGreens(greens_cfg1(), prec)
    pp, vv = (p, v) if prec else (p.astype(np.float32), v.astype(np.float32))
    for law, kir, sc in ((0, 0, 1.0), (1, 0, 0.25), (1, 1, 0.15)):
        base = None
        for k0 in (0, 5, -1, -2, -3, -4):
            out, it, st, _, ms = dg.fp_batch_host(pp * sc, vv, dg.fp_opts(leak_frac=0.3, beta=0.017, law=law, kirchhoff=kir,
                                                                          tol=1e-4, max_iters=200, accel=k0))
            out, it, st, _, ms = dg.fp_batch_host(pp * sc, vv, dg.fp_opts(leak_frac=0.3, beta=0.017, law=law, kirchhoff=kir,
                                                                          tol=1e-4, max_iters=200, accel=k0))
            if base is None:
                base = out
            print(f"prec={'fp64' if prec else 'fp32'} law={law} kir={kir} accel={k0}: mean iters {it.mean():.2f} max {it.max()} "
                  f"failed {(st != 0).sum()} max|dT| vs Picard {np.abs(out - base).max():.2e} K  online {ms:.1f} ms", flush=True)
    dg.close()

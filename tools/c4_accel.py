"""Config 4 on one GPU at 300 W: Picard, Chebyshev (accel 3) and low-mode Anderson (accel -m)."""
import ctypes as C
import dataclasses
import sys
import tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2307_12119_b200 import inputs, slab
from paper_2307_12119_b200.api import DeviceGreens, GreensArrays, lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = Path(tempfile.mkdtemp())
(d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
f = np.empty((n, n))
nn = C.c_int()
L = lib()
assert L.gt_modal_kernel(str(d / "stack.txt").encode(), C.byref(nn), f.ctypes.data_as(C.POINTER(C.c_double))) == 0
phi = float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]])))
ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=f, phi=phi, kappa_inf=float(f[0, 0]), alpha=0.0,
                  beta=0.017, mu=0.0, rand_scale=1.0)
dg = DeviceGreens(ga, 1)
cfg = dataclasses.replace(inputs.CONFIGS["cfg4"], n=n)
P = inputs.power_map_torch(cfg, 0, device="cuda")
P *= 300.0 / float(P.sum())
V = inputs.variation_batch(cfg, 0, 1, device="cuda", dtype=torch.float64)[0]
ops = slab.GpuLargeOps(dg)
base = None
for accel in (0, 3, -2, -3, -4):
    o = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
    o.accel = accel
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = slab.solve_slab(ops, n, P, V, o)
        e1.record()
        torch.cuda.synchronize()
    if base is None:
        base = res.t.clone()
    print(f"accel {accel}: {e0.elapsed_time(e1):.1f} ms, {res.iterations} iterations, status {res.status}, "
          f"max|dT| vs Picard {float((res.t - base).abs().max()):.2e} K, peak {float(res.t.max()):.1f} K", flush=True)

"""Config-4 timing on one GPU: n x n map (default 8192), mode-B linear law to 1e-4 K, fp64."""
import ctypes as C
import sys
import tempfile
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2307_12119_b200 import inputs, slab
from paper_2307_12119_b200.api import DeviceGreens, GreensArrays, lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
t0 = time.time()
d = Path(tempfile.mkdtemp())
(d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
f = np.empty((n, n))
nn = C.c_int()
L = lib()
assert L.gt_modal_kernel(str(d / "stack.txt").encode(), C.byref(nn), f.ctypes.data_as(C.POINTER(C.c_double))) == 0
t1 = time.time()
phi = float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]])))
ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=f, phi=phi, kappa_inf=float(f[0, 0]), alpha=0.0,
                  beta=0.017, mu=0.0, rand_scale=1.0)
dg = DeviceGreens(ga, 1)
t2 = time.time()
cfg = inputs.CONFIGS["cfg4"]
import dataclasses
cfg = dataclasses.replace(cfg, n=n)
P = torch.from_numpy(inputs.power_map(cfg, 0)).cuda()
V = inputs.variation_batch(cfg, 0, 1, device="cuda", dtype=torch.float64)[0]
t3 = time.time()
print(f"modal kernel {t1 - t0:.1f} s, prepare {t2 - t1:.1f} s, inputs {t3 - t2:.1f} s; P total {P.sum().item():.1f} W")
ops = slab.GpuLargeOps(dg)
o = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=200)
o2 = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=0, tol=1e-4, max_iters=2)
slab.solve_slab(ops, n, P, V, o2)
torch.cuda.synchronize()
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = slab.solve_slab(ops, n, P, V, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    h = n + 1
    b_it = 5 * 8 * n * n + 8 * 8 * n * h
    print(f"rep {rep}: {ms:.1f} ms, {res.iterations} iterations ({ms / res.iterations:.2f} ms/it), status {res.status}, "
          f"peak {res.t.max().item():.2f} K, model {b_it * res.iterations / (ms / 1e3) / 1e9:.0f} GB/s")

"""Config-2 combined solve (n = 1024: shift-variant + Kirchhoff + exp-law loop, fp32 with the fp64
finish) for an ncu launch list. usage: python tools/prof_cfg2c.py [B] [scale]"""
import ctypes as C
import sys
import tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import GT_FP32, DeviceGreens, GreensArrays, lib

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.15
n = 1024
d = Path(tempfile.mkdtemp())
(d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
f = np.empty((n, n))
nn = C.c_int()
assert lib().gt_modal_kernel(str(d / "stack.txt").encode(), C.byref(nn), f.ctypes.data_as(C.POINTER(C.c_double))) == 0
phi = float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]])))
ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=f, phi=phi, kappa_inf=float(f[0, 0]), alpha=1e-3,
                  beta=0.017, mu=0.0, rand_scale=1.0)
P, V = inputs.mc_inputs(inputs.CONFIGS["cfg2"], 0, B, device="cuda", torch_dtype=torch.float32)
P = (P * scale).contiguous()
dg = DeviceGreens(ga, GT_FP32)
T = torch.empty_like(P)
it = torch.zeros(B, dtype=torch.int32, device="cuda")
st = torch.zeros(B, dtype=torch.int32, device="cuda")
fo = dg.fp_opts(leak_frac=0.3, beta=0.017, law=1, kirchhoff=1, with_rand=1, tol=1e-4, max_iters=200)
s = torch.cuda.Stream()
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    dg.fp_batch_device(P.data_ptr(), V.data_ptr(), B, fo, T.data_ptr(), it.data_ptr(), st.data_ptr(), None, None,
                       s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"B={B}: {e0.elapsed_time(e1):.2f} ms, iterations {it.float().mean().item():.2f}, "
          f"failed {(st != 0).sum().item()}", flush=True)

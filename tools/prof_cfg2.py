"""Config-2 grid (n = 1024) workload for timing / ncu: mode A fp32 and mode B fp64 (Kirchhoff).

usage: python tools/prof_cfg2.py [B] [modeB_iters]
The kernel comes from gt_modal_kernel (alpha = 0): the pass costs do not depend on it.
"""
import ctypes as C
import sys
import tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import GT_FP32, GT_FP64, SAMPLE_STATS_DTYPE, DeviceGreens, GreensArrays, lib

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = 1024
d = Path(tempfile.mkdtemp())
(d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
f = np.empty((n, n))
nn = C.c_int()
assert lib().gt_modal_kernel(str(d / "stack.txt").encode(), C.byref(nn), f.ctypes.data_as(C.POINTER(C.c_double))) == 0
phi = float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]])))
ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=f, phi=phi, kappa_inf=float(f[0, 0]), alpha=0.0,
                  beta=0.017, mu=0.0, rand_scale=1.0)
cfg = inputs.CONFIGS["cfg2"]
P, V = inputs.mc_inputs(cfg, 0, B, device="cuda", torch_dtype=torch.float32)
s = torch.cuda.Stream()

dg = DeviceGreens(ga, GT_FP32)
out = torch.empty_like(P)
st = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
for rep in range(3):
    dg.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    dg.mc_batch_device(P.data_ptr(), V.data_ptr(), B, dg.opts(), out.data_ptr(), st.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    pm, k, c = dg.profile_end()
    print(f"mode A fp32 B={B}: {e0.elapsed_time(e1):.2f} ms, passes {[round(x, 3) for x in pm[:3]]} ms")
dg.close()

P64 = (P.double() * 0.3).contiguous()
V64 = V.double().contiguous()
dg = DeviceGreens(ga, GT_FP64)
fo = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=1, tol=1e-30, max_iters=iters)
T = torch.empty_like(P64)
it = torch.zeros(B, dtype=torch.int32, device="cuda")
sd = torch.zeros(B, dtype=torch.int32, device="cuda")
mx = torch.zeros(B, dtype=torch.float64, device="cuda")
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    dg.fp_batch_device(P64.data_ptr(), V64.data_ptr(), B, fo, T.data_ptr(), it.data_ptr(), sd.data_ptr(),
                       mx.data_ptr(), None, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"mode B fp64 B={B}: {e0.elapsed_time(e1):.2f} ms for {iters} iterations "
          f"({e0.elapsed_time(e1) / iters:.2f} ms/it)")
dg.close()
print("done")

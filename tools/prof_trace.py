"""Config-3 timing: B traces x steps at n (device-calibrated GreensSet)."""
import ctypes as C
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens, GreensArrays, lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 0


def greens(n):
    import tempfile
    L = lib()
    d = Path(tempfile.mkdtemp())
    (d / "stack.txt").write_text(f"n {n}\ndie_edge 0.016\n")
    (d / "var.txt").write_text("dopant_spread 0\nbeta 0.017\n")
    g = C.c_void_p()
    assert L.gt_calibrate(str(d / "stack.txt").encode(), str(d / "var.txt").encode(), None, 90.0, C.byref(g),
                          None) == 0, L.gt_last_error()
    maps = {}
    for k in ("f_sp0", "g_sp0"):
        f = C.c_void_p()
        assert L.gt_greens_field(g, k.encode(), C.byref(f)) == 0
        maps[k] = np.ctypeslib.as_array(L.gt_field_data(f), shape=(n, n)).copy()
        L.gt_field_free(f)
    f = maps["f_sp0"]
    ga = GreensArrays(n=n, pitch=0.016 / n, f_sp0=f, g_sp0=maps["g_sp0"],
                      phi=float(np.mean(np.concatenate([f[0], f[-1], f[1:-1, 0], f[1:-1, -1]]))),
                      kappa_inf=float(f[0, 0]), alpha=L.gt_greens_alpha(g), beta=0.017, mu=L.gt_greens_mu(g),
                      capacitance=L.gt_greens_capacitance(g), rand_scale=1.0)
    L.gt_greens_free(g)
    return ga


t0 = time.time()
ga = greens(n)
print(f"calibrated n={n} in {time.time() - t0:.1f} s, capacitance {ga.capacitance:.3e}")
cfg = inputs.CONFIGS["cfg3"]
import dataclasses
cfg = dataclasses.replace(cfg, n=n)
blks, scheds, ons = zip(*(inputs.markov_blocks(cfg, b, steps) for b in range(B)))
nblk = max(s.shape[1] for s in scheds)
sched = np.zeros((B, steps, nblk))
for b, s in enumerate(scheds):
    sched[b, :, :s.shape[1]] = s
dt_t = torch.float64 if prec else torch.float32
var = inputs.variation_batch(cfg, 0, B, device="cuda", dtype=dt_t)
leak0 = torch.from_numpy(0.3 * np.stack(ons)).to(dt_t).cuda() * var
blk = torch.from_numpy(np.stack(blks)).cuda()
sch = torch.from_numpy(sched).to(dt_t).cuda()
dg = DeviceGreens(ga, prec)
stride = 100 if steps >= 100 else 1
frames = steps // stride
out = torch.zeros((B, frames, n, n), dtype=dt_t, device="cuda")
mx = torch.zeros((B, frames), dtype=torch.float64, device="cuda")
o = dg.trace_opts(dt=1e-5, steps=steps, window=500, law=0, beta=0.017, out_stride=stride)
s = torch.cuda.Stream()
for rep in range(int(sys.argv[5]) if len(sys.argv) > 5 else 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    dg.trace_batch_device(blk.data_ptr(), n * n, sch.data_ptr(), nblk, leak0.data_ptr(), n * n, B, o,
                          out.data_ptr(), mx.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"rep {rep}: {ms:.1f} ms for {B} traces x {steps} steps = {B * steps / ms * 1e3:.0f} trace-steps/s "
          f"({ms / steps * 1e3:.1f} us per step); peak T {mx.max().item():.2f} K")

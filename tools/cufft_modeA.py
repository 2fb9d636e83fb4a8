"""Library baseline for the headline (measurement only, NOT a product path): config-1
mode A (reference run_one with gs.mu closed forms, solver.cpp:353-374, greens.cpp:203-251)
written with torch + cuFFT (rfft2 / irfft2 of the 2n-padded maps, the closed forms as
elementwise torch ops) on the same pairs, timed with CUDA events next to the product's
fused passes, and checked against them.
argv: [pairs=4096] [chunk=512] [precision fp32|fp64]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import GT_FP32, GT_FP64, DeviceGreens, SAMPLE_STATS_DTYPE

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
CH = int(sys.argv[2]) if len(sys.argv) > 2 else 512
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
dt, cdt = (torch.float32, torch.complex64) if prec == "fp32" else (torch.float64, torch.complex128)
dev = "cuda"
g = greens_cfg1()
n, m, c = g.n, 2 * g.n, g.n // 2
h = n + 1
LEAK = 0.3


def center(x):  # center_kernel (spectral.cpp:126-141): K[(i - c) mod m][(j - c) mod m] = x[i][j]
    out = torch.zeros(x.shape[:-2] + (m, m), dtype=x.dtype, device=x.device)
    out[..., :n, :n] = x
    return torch.roll(out, shifts=(-c, -c), dims=(-2, -1))


def symmetric_multiplier_half(x):  # spectral.cpp:167-185 on the half plane j <= n
    i = torch.arange(m, device=dev)
    dx = torch.minimum(i, m - i)
    dy = torch.arange(h, device=dev)
    ip, im = (c + dx).clamp(0, n - 1), (c - dx).clamp(0, n - 1)
    jp, jm = (c + dy).clamp(0, n - 1), (c - dy).clamp(0, n - 1)
    g_ = lambda a, b: x[..., a[:, None], b[None, :]]
    return 0.25 * (g_(ip, jp) + g_(ip, jm) + g_(im, jp) + g_(im, jm))


# ---- per-GreensSet spectra (fp64, once): fk, alpha multiplier, F_det at gs.mu
f = torch.from_numpy(g.f_sp0).to(dev)
fk = torch.fft.fft2(center(f - g.phi))
fk[0, 0] += g.phi * m * m / 4  # baseline_kernel_spectrum (greens.cpp:194-201)
gsp = torch.from_numpy(g.g_sp0).to(dev)
gm = gsp[c, c] - symmetric_multiplier_half(gsp)  # alpha_multiplier on the half plane
fkh = fk[:, :h]
den1 = 1.0 - g.alpha * gm - g.mu * g.beta * fkh  # F(mu) only touches DC, where g = 0
fdet = (fkh / den1).to(cdt)
fkh_c, gm_c = fkh.to(cdt), gm.to(dt)


def solve(P, V):
    L = LEAK * P * V
    app = P + L
    mu_s = L.mean(dim=(-2, -1), keepdim=True)
    pvar = L - mu_s
    mir = torch.cat([app, app.flip(-2)], -2)
    mir = torch.cat([mir, mir.flip(-1)], -1)
    tdet = torch.fft.irfft2(torch.fft.rfft2(mir) * fdet, s=(m, m))[..., :n, :n]
    q = symmetric_multiplier_half(pvar) + (pvar[..., c:c + 1, c:c + 1] - pvar[..., 0:1, 0:1])  # q_rand shift
    fpv = torch.fft.rfft2(center(pvar))
    t1 = g.beta * fkh_c * q + g.alpha * gm_c * fpv
    frand = fdet * t1 / (den1.to(cdt) - t1)
    fr = torch.roll(torch.fft.irfft2(frand, s=(m, m)), shifts=(c, c), dims=(-2, -1))[..., :n, :n]  # kernel_to_die
    tot = app.sum(dim=(-2, -1), keepdim=True) * g.rand_scale
    return torch.clamp(tdet + fr * pvar * tot, min=0.0)


cfg = inputs.CONFIGS["cfg1"]
P, V = inputs.mc_inputs(cfg, 0, B, device=dev, torch_dtype=dt)
out = torch.empty_like(P)
for _ in range(2):  # warm-up (cuFFT plans)
    out[:CH] = solve(P[:CH], V[:CH])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for s0 in range(0, B, CH):
    out[s0:s0 + CH] = solve(P[s0:s0 + CH], V[s0:s0 + CH])
e1.record()
torch.cuda.synchronize()
ms_lib = e0.elapsed_time(e1)
# the product on the same pairs
dg = DeviceGreens(g, GT_FP32 if prec == "fp32" else GT_FP64)
o2 = torch.empty_like(P)
st = torch.zeros(B * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device=dev)
opts = dg.opts(leak_frac=LEAK, mu_per_sample=0, with_rand=1)
for _ in range(2):
    dg.mc_batch_device(P.data_ptr(), V.data_ptr(), B, opts, o2.data_ptr(), st.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
e0.record()
dg.mc_batch_device(P.data_ptr(), V.data_ptr(), B, opts, o2.data_ptr(), st.data_ptr(), torch.cuda.current_stream().cuda_stream)
e1.record()
torch.cuda.synchronize()
ms_prod = e0.elapsed_time(e1)
d = (out.double() - o2.double()).abs().reshape(B, -1).amax(1)
print(f"{prec}, {B} pairs: torch+cuFFT {ms_lib:.2f} ms ({B / ms_lib * 1e3:.0f} solves/s), "
      f"product {ms_prod:.2f} ms ({B / ms_prod * 1e3:.0f} solves/s): {ms_lib / ms_prod:.2f}x; "
      f"max |dT| between them {float(d.max()):.3e} K (median pair {float(d.median()):.2e})")

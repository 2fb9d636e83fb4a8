"""fp32 vs fp64 of mode A on the bench's pairs, per closed-form mu semantics, next to each
pair's conditioning max 1/|den2|^2 (stats.max_rden2)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens, SAMPLE_STATS_DTYPE

K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = inputs.CONFIGS["cfg1"]
P, V = inputs.mc_inputs(cfg, 0, K, device="cuda", torch_dtype=torch.float32)
res, rd = {}, {}
for prec in (0, 1):
    dg = DeviceGreens(greens_cfg1(), prec)
    p = P.double().contiguous() if prec else P
    v = V.double().contiguous() if prec else V
    for mps in (0, 1):
        out = torch.empty_like(p)
        st = torch.zeros(K * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        dg.mc_batch_device(p.data_ptr(), v.data_ptr(), K, dg.opts(mu_per_sample=mps), out.data_ptr(), st.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        s = np.frombuffer(st.cpu().numpy().tobytes(), dtype=SAMPLE_STATS_DTYPE)
        res[(prec, mps)] = out.double().cpu().numpy()
        rd[(prec, mps)] = s["max_rden2"].copy()
    dg.close()
for mps in (0, 1):
    e = np.abs(res[(0, mps)] - res[(1, mps)]).reshape(K, -1).max(1)
    r = rd[(1, mps)]
    o = np.argsort(-e)[:8]
    print(f"mu_per_sample={mps}: fp32 vs fp64 max {e.max():.3e} K; pairs > 1e-3 K: {(e > 1e-3).sum()} of {K}; "
          f"> 5e-4: {(e > 5e-4).sum()}")
    print("   worst pairs (err, max 1/|den2|^2 fp64, fp32):", [(int(i), f"{e[i]:.2e}", f"{r[i]:.3g}",
                                                               f"{rd[(0, mps)][i]:.3g}") for i in o])
    print("   rden2 quantiles:", np.quantile(r, [0.5, 0.9, 0.99, 1.0]))
    for thr in (1e2, 1e3, 1e4, 1e5, 1e6):
        sel = rd[(0, mps)] > thr
        print(f"   thr {thr:.0e}: {sel.sum()} pairs flagged; max err unflagged {e[~sel].max() if (~sel).any() else 0:.2e}")

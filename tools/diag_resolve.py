"""fp32 (no re-solve) vs fp64 of mode A (gs.mu semantics) on K config-1 pairs: per-pair max
error next to the pair's conditioning statistic stats.max_rden2 (max 1/|den2|^2), to set the
fp64 re-solve threshold. argv: K tag -> gpurun_out/diag_<tag>.npz;
`python tools/diag_resolve.py analyse tag...` prints flagged counts vs max unflagged error.
(An alternative statistic, max |F_rand|^2 (alpha g)^2 / |den2|^2, was tried as a compile-time
variant and correlated far worse: profiles/r2s2_ncu_summary.md.)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

if sys.argv[1] == "analyse":
    A = [np.load(f"gpurun_out/diag_{t}.npz") for t in sys.argv[2:]]
    err = A[0]["err"]
    print(f"{len(err)} pairs; err max {err.max():.3e}; > 1e-3: {(err > 1e-3).sum()}, > 5e-4: {(err > 5e-4).sum()}")
    for t, a in zip(sys.argv[2:], A):
        for scale in (False, True):
            s = a["stat"] * (a["sumapp"] ** 2 if scale else 1.0)
            print(f"-- {t} {'x sum^2' if scale else ''}")
            for q in (0.9, 0.95, 0.98, 0.99, 0.995, 0.998, 0.999):
                thr = np.quantile(s, q)
                sel = s > thr
                print(f"   flag top {100 * (1 - q):.1f}% ({sel.sum()}): max err unflagged {err[~sel].max():.2e}")
    sys.exit(0)

import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import GT_FP32, GT_FP64, DeviceGreens, SAMPLE_STATS_DTYPE

K, tag = int(sys.argv[1]), sys.argv[2]
cfg = inputs.CONFIGS["cfg1"]
CH = 512
d32, d64 = DeviceGreens(greens_cfg1(), GT_FP32), DeviceGreens(greens_cfg1(), GT_FP64)
errs, stats, sums = [], [], []
for s0 in range(0, K, CH):
    P, V = inputs.mc_inputs(cfg, s0, CH, device="cuda", torch_dtype=torch.float32)
    o32 = torch.empty_like(P)
    st = torch.zeros(CH * SAMPLE_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    d32.mc_batch_device(P.data_ptr(), V.data_ptr(), CH, d32.opts(mu_per_sample=0, fp64_check=-1.0), o32.data_ptr(),
                        st.data_ptr(), torch.cuda.current_stream().cuda_stream)
    P64, V64 = P.double(), V.double()
    o64 = torch.empty_like(P64)
    st64 = torch.zeros_like(st)
    d64.mc_batch_device(P64.data_ptr(), V64.data_ptr(), CH, d64.opts(mu_per_sample=0), o64.data_ptr(),
                        st64.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    errs.append((o32.double() - o64).abs().reshape(CH, -1).amax(1).cpu().numpy())
    s = np.frombuffer(st.cpu().numpy().tobytes(), dtype=SAMPLE_STATS_DTYPE)
    stats.append(s["max_rden2"].astype(np.float64))
    sums.append(s["sum_applied"].copy())
np.savez(f"gpurun_out/diag_{tag}.npz", err=np.concatenate(errs), stat=np.concatenate(stats),
         sumapp=np.concatenate(sums))
print("saved", tag)

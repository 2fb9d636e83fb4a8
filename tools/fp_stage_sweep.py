"""Mode B (config 1, linear law, 1e-4 K) on an fp32 handle: the fp32 stage tolerance
(gt_fp_opts.fp32_stage_tol; the fp64 finish iterates from there to 1e-4 K) and Chebyshev
start vs time, mean iterations and the distance to the fp64-handle Picard fixed point."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import greens_cfg1
from paper_2307_12119_b200 import inputs
from paper_2307_12119_b200.api import DeviceGreens

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = inputs.CONFIGS["cfg1"]
P, V = inputs.mc_inputs(cfg, 0, B, device="cuda", torch_dtype=torch.float32)
it = torch.zeros(B, dtype=torch.int32, device="cuda")
st = torch.zeros(B, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
d64 = DeviceGreens(greens_cfg1(), 1)
P64, V64 = P.double(), V.double()
T64 = torch.empty_like(P64)
d64.fp_batch_device(P64.data_ptr(), V64.data_ptr(), B, d64.fp_opts(leak_frac=0.3, law=0, kirchhoff=0, beta=0.017,
                    tol=1e-4, max_iters=200), T64.data_ptr(), it.data_ptr(), st.data_ptr(), None, None, s)
torch.cuda.synchronize()
print(f"fp64 Picard reference: mean iterations {it.double().mean():.2f}")
d64.close()
del P64, V64
d = DeviceGreens(greens_cfg1(), 0)
T = torch.empty_like(P)
for accel in ([int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else (0, 5)):
    for tol32 in [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("5e-4", "3e-4", "2e-4", "1.5e-4"))]:
        o = d.fp_opts(leak_frac=0.3, law=0, kirchhoff=0, beta=0.017, tol=1e-4, max_iters=200, accel=accel,
                      fp32_stage_tol=tol32)
        d.fp_batch_device(P.data_ptr(), V.data_ptr(), B, o, T.data_ptr(), it.data_ptr(), st.data_ptr(), None, None, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            d.fp_batch_device(P.data_ptr(), V.data_ptr(), B, o, T.data_ptr(), it.data_ptr(), st.data_ptr(), None, None, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        err = float((T.double() - T64).abs().max())
        print(f"accel {accel} fp32_stage_tol {tol32:.1e}: {B / ms * 1e3:.0f} solves/s, mean iterations "
              f"{it.double().mean():.2f} (max {int(it.max())}), failed {int((st != 0).sum())}, "
              f"max |dT| vs fp64 Picard {err:.2e} K", flush=True)

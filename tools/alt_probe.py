import sys, time
sys.argv = ["x", "64", "4"]
exec(open("tools/prof_cfg2.py").read().split("P64 = ")[0].replace("for rep in range(3):", "for rep in range(0):"))
import torch
from paper_2307_12119_b200.api import GT_FP64, DeviceGreens
P64 = (P.double() * 0.3).contiguous(); V64 = V.double().contiguous()
dg = DeviceGreens(ga, GT_FP64)
T = torch.empty_like(P64)
it = torch.zeros(B, dtype=torch.int32, device="cuda"); sd = torch.zeros_like(it); mx = torch.zeros(B, dtype=torch.float64, device="cuda")
for kir in ((1,) if len(sys.argv) > 9 else (1, 0)):
    fo = dg.fp_opts(leak_frac=0.3, beta=0.017, law=0, kirchhoff=kir, tol=1e-30, max_iters=4)
    for rep in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        dg.fp_batch_device(P64.data_ptr(), V64.data_ptr(), B, fo, T.data_ptr(), it.data_ptr(), sd.data_ptr(), mx.data_ptr(), None, s.cuda_stream)
        e1.record(s)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"kirchhoff={kir} rep {rep}: dev {e0.elapsed_time(e1):.2f} ms, host call {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms")

import torch, time
for mb in (32, 256, 1024):
    n = mb * 2**20 // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"H2D {mb} MiB chunks: {5*mb*2**20/e0.elapsed_time(e1)/1e6:.1f} GB/s")

import torch
# one stream vs two streams of concurrent H2D copies (aggregate PCIe rate)
mb = 1024
n = mb * 2**20 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d.copy_(h, non_blocking=True); torch.cuda.synchronize()
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(3):
        for k, s in enumerate(ss):
            s.wait_event(e0) if it == 0 else None
            with torch.cuda.stream(s):
                part = n // ns
                d[k*part:(k+1)*part].copy_(h[k*part:(k+1)*part], non_blocking=True)
    for s in ss:
        ev = torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
    e1.record(); torch.cuda.synchronize()
    print(f"H2D 1 GiB x3 over {ns} stream(s): {3*mb*2**20/e0.elapsed_time(e1)/1e6:.1f} GB/s")

import torch, time
n = 2 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device='cuda')
s = torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(3): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, 3 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, "GB/s")

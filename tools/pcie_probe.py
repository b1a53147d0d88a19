import torch, time
x = torch.empty(217_000_000, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
z = torch.empty(67_000_000, dtype=torch.uint8).pin_memory()
w = torch.empty_like(z, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
for label, fn in [("h2d 217MB", lambda: y.copy_(x, non_blocking=True)), ("d2h 67MB", lambda: z.copy_(w, non_blocking=True))]:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/10
    print(label, ms, "ms", (217e6 if 'h2d' in label else 67e6)/ms/1e6, "GB/s")

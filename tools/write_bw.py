import torch
x = torch.empty(1 << 30, dtype=torch.int64, device="cuda")
y = torch.empty(1 << 30, dtype=torch.int64, device="cuda")
for name, fn in [("fill", lambda: x.fill_(7)), ("copy", lambda: y.copy_(x))]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    b = 8 * (1 << 30) * (1 if name == "fill" else 2)
    print(name, ms, "ms", b / ms / 1e6, "GB/s")

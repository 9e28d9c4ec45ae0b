import torch, time
x = torch.empty(275_000_000, dtype=torch.int32, device="cuda")
h = torch.empty_like(x, device="cpu").pin_memory()
for i in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); h.copy_(x, non_blocking=True); e.record(); torch.cuda.synchronize()
    print("D2H 1.1GB ms", s.elapsed_time(e), "GB/s", 1.1e9 / s.elapsed_time(e) / 1e6)
for i in range(2):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); x.copy_(h, non_blocking=True); e.record(); torch.cuda.synchronize()
    print("H2D 1.1GB ms", s.elapsed_time(e))

import time, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2009_06693_b200.graph import device_view
x = torch.empty(275_000_000, dtype=torch.int32, device="cuda")
v = device_view(x.data_ptr(), x.numel(), "int32", x)
h = torch.empty(x.numel(), dtype=torch.int32, pin_memory=True)
hb = h[: x.numel() - 5]
cs = torch.cuda.Stream()
for src, dst, name in ((x, h, "torch->pinned"), (v, h, "view->pinned"), (v[: x.numel() - 5], hb, "view slice->pinned slice")):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(cs):
        dst.copy_(src, non_blocking=True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(name, "pinned", dst.is_pinned(), "enqueue ms", round((t1 - t0) * 1e3, 3), "total ms", round((t2 - t0) * 1e3, 3))

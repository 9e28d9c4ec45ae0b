"""Dev probe: does a concurrent device->host copy slow the walk kernel?"""
import sys, os, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
app = make_app("node2vec")
V = dg.n_vertices
src = torch.empty(275_000_000, dtype=torch.int32, device="cuda")
dst_h = torch.empty(src.numel(), dtype=torch.int32, pin_memory=True)
dst_d = torch.empty_like(src)
cs = torch.cuda.Stream()
run_device(app, dg, n_samples=V, seed=7, paradigm="sp").close()
for mode in ("alone", "d2h", "d2d", "h2d", "alone"):
    ms = []
    for it in range(3):
        torch.cuda.synchronize()
        if mode != "alone":
            with torch.cuda.stream(cs):
                for _ in range(3):  # ~60 ms of copies, longer than the walk
                    if mode == "d2h": dst_h.copy_(src, non_blocking=True)
                    elif mode == "d2d": dst_d.copy_(src, non_blocking=True)
                    else: src.copy_(dst_h, non_blocking=True)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dr = run_device(app, dg, n_samples=V, seed=7, paradigm="sp")
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
        dr.close()
    print(mode, round(statistics.median(ms), 2), flush=True)

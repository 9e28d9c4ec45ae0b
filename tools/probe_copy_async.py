"""Dev probe: is nd_result_copy into the pipeline's pinned buffers host-asynchronous?"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app, _lib  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
g = DeviceGraph.rmat(20, n_edges=17_000_000, seed=0, weighted=True)
dr = run_device(make_app("deepwalk"), g, n_samples=1 << 20, seed=7, paradigm="sp")
L = _lib.load()
cs = torch.cuda.Stream()
for pin in (True, False):
    n = dr.field_count(_lib.F_FINAL_IDS32)[1]
    h = torch.empty(n, dtype=torch.int32, pin_memory=pin)
    hv = h[:n]
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(L.nd_result_copy(dr._h, _lib.F_FINAL_IDS32, _lib.ptr(hv), _lib.stream_ptr(cs)), "copy")
        t1 = time.perf_counter()
        cs.synchronize()
        t2 = time.perf_counter()
        print(f"pinned={pin} bytes={n*4} call_ms={1e3*(t1-t0):.3f} total_ms={1e3*(t2-t0):.3f}", flush=True)

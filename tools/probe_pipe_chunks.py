"""Dev probe: node2vec chunk compute time with and without the previous
chunk's D2H in flight (single job, events on the compute stream)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app, _lib  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
V = dg.n_vertices
L = _lib.load()
for name in ("node2vec", "ppr"):
    app = make_app(name)
    C = 6
    step = V // C
    st, cs = torch.cuda.Stream(), torch.cuda.Stream()
    bufs = [torch.empty(200_000_000, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    for copy in (False, True, False, True):
        prev = None
        comp = []
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            for c in range(C):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                dr = run_device(app, dg, n_samples=step, sample_lo=c * step, seed=7, paradigm="sp",
                                stream=st, sync=False)
                e1.record(st)
                if copy:
                    ready = torch.cuda.Event()
                    ready.record(st)
                    cs.wait_event(ready)
                    n = dr.field_count(_lib.F_FINAL_IDS32)[1]
                    _lib.check(L.nd_result_copy(dr._h, _lib.F_FINAL_IDS32, _lib.ptr(bufs[c % 2][:n]),
                                                _lib.stream_ptr(cs)), "copy")
                comp.append((e0, e1))
                if prev is not None:
                    prev.close()
                prev = dr
        torch.cuda.synchronize()
        prev.close()
        print(name, "copy" if copy else "nocopy", [round(a.elapsed_time(b), 2) for a, b in comp],
              "total", round(comp[0][0].elapsed_time(comp[-1][1]), 2), flush=True)

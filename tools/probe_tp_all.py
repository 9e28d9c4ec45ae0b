"""Dev probe: TP timings for C2 walks (class kernels only) and C3 k-hop."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
def t(app, g, n, par, reps=3):
    ms = []
    for _ in range(reps + 1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dr = run_device(app, g, n_samples=n, seed=7, paradigm=par); e.record()
        torch.cuda.synchronize(); ms.append(s.elapsed_time(e)); dr.close()
    return statistics.median(ms[1:])
g2 = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
for tail in ("0", "131072"):
    os.environ["ND_TP_TAIL"] = tail
    for name in ("node2vec", "ppr"):
        print(f"C2 {name} TP tail={tail}: {t(make_app(name), g2, g2.n_vertices, 'tp'):.2f} ms", flush=True)
g2.close()
g3 = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
print(f"C3 khop TP: {t(make_app('khop'), g3, 233472, 'tp'):.3f} ms  SP: {t(make_app('khop'), g3, 233472, 'sp'):.3f} ms", flush=True)

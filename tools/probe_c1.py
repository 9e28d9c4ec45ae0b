"""Dev probe: C1 DeepWalk (PPI-shaped powerlaw, L2-resident), median event time;
argv[1]: paradigm (sp | tp)."""
import sys, os, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.synth import powerlaw_graph  # noqa: E402
g = powerlaw_graph(56944, attach=7, weighted=True, seed=0)
dg = DeviceGraph.from_graph(g)
app = make_app("deepwalk")
ms = []
for it in range(12):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    dr = run_device(app, dg, n_samples=dg.n_vertices, seed=7, paradigm=sys.argv[1] if len(sys.argv) > 1 else "sp")
    e.record(); torch.cuda.synchronize()
    if it > 1: ms.append(s.elapsed_time(e))
    dr.close()
print("C1 deepwalk", sys.argv[1:] or ["sp"], "ms", round(statistics.median(ms), 4))

"""Dev probe: C3 k-hop device-only timing per paradigm (ND_TRACE=1 for phases)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
app = make_app("khop")
N = 1024 * 228
for par in sys.argv[1:] or ["tp", "sp"]:
    for it in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par)
        e.record()
        torch.cuda.synchronize()
        print(par, it, s.elapsed_time(e), dr.total_sampled, flush=True)
        dr.close()

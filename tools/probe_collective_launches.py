"""Dev probe: one C4 collective run (default ClusterGCN) inside cudaProfilerStart/Stop
for an ncu launch list; also prints event-timed ms for TP and SP."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "clustergcn"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kw = {"distribution": "degree_sq"} if name == "ladies" else {}
dg = DeviceGraph.rmat(22, n_edges=58_600_000, seed=0, undirected=True, weighted=False)
app = make_app(name, **kw)
for par in ("tp", "sp"):
    for it in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par); e.record()
        torch.cuda.synchronize(); dr.close()
    print(name, par, "ms", s.elapsed_time(e), flush=True)
torch.cuda.cudart().cudaProfilerStart()
run_device(app, dg, n_samples=N, seed=7, paradigm="tp").close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

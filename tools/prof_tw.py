"""Dev probe for ncu: one C2 TP (hub engine) run of an app after a warm-up run."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "deepwalk"
kw = {"node2vec": {"p": 2.0, "q": 0.5}, "ppr": {"termination_probability": 0.01}}.get(name, {})
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 22
g = DeviceGraph.rmat(scale, n_edges=68_993_773 if scale == 22 else 16 << scale, seed=0, weighted=True)
app = make_app(name, **kw)
os.environ["ND_TP_TAIL"] = os.environ.get("ND_TP_TAIL", "131072")
run_device(app, g, n_samples=g.n_vertices, seed=7, paradigm="sp").close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
dr = run_device(app, g, n_samples=g.n_vertices, seed=7, paradigm="tp")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
st = dr.host(10).reshape(-1, 4) if dr.host(10) is not None else None
print("steps", dr.n_steps, "edges", dr.total_sampled)
if st is not None:
    for s in (0, 1, 2, 10, 50, 99):
        if s < len(st):
            print("step", s, "small/med/large/groups", st[s].tolist())
dr.close()

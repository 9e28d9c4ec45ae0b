"""Dev probe for ncu: one C4 ClusterGCN run, one C4 FastGCN run and one TP
node2vec step window (C2) inside cudaProfilerStart/Stop."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
which = sys.argv[1]
if which in ("clustergcn", "fastgcn"):
    g = DeviceGraph.rmat(22, n_edges=58_600_000, seed=0, undirected=True, weighted=False)
    app, n, par = make_app(which), (8 if which == "clustergcn" else 4096), "tp"
else:
    g = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
    app, n, par = make_app("node2vec", p=2.0, q=0.5, walk_length=3), g.n_vertices, "tp"
    os.environ["ND_TP_TAIL"] = "0"
run_device(app, g, n_samples=n, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run_device(app, g, n_samples=n, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

"""One C2 node2vec TP run inside cudaProfilerStart/Stop (ncu target for the
TP walk engine's kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
app = make_app(sys.argv[1] if len(sys.argv) > 1 else "node2vec")
run_device(app, dg, n_samples=dg.n_vertices, seed=7, paradigm="tp").close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run_device(app, dg, n_samples=dg.n_vertices, seed=7, paradigm="tp").close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

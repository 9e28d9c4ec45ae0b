"""One C3 k-hop TP run inside cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
app = make_app("khop", fanouts=[25, 10])
par = sys.argv[1] if len(sys.argv) > 1 else "tp"
run_device(app, dg, n_samples=1024 * 228, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run_device(app, dg, n_samples=1024 * 228, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

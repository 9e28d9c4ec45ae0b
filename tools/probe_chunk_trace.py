"""Dev probe: ND_TRACE phase timeline of one node2vec / PPR chunk (700K walkers)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
g = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
for app in (make_app("node2vec", p=2.0, q=0.5), make_app("ppr", termination_probability=0.01)):
    for it in range(3):
        if it == 2:
            print("----", app.name, file=sys.stderr, flush=True)
            os.environ["ND_TRACE"] = "1"
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dr = run_device(app, g, n_samples=699050, sample_lo=699050, seed=7, paradigm="sp")
        e.record(); torch.cuda.synchronize()
        dr.close()
        os.environ.pop("ND_TRACE", None)
    print(app.name, "ms", s.elapsed_time(e), file=sys.stderr, flush=True)

"""Dev probe: per-chunk cost of the host pipeline, one app at a time, no copies."""
import os, sys, statistics
os.environ["ND_PIPE_NOCOPY"] = "1"
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.streaming import HostPipeline  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
V = dg.n_vertices
for app in (make_app("node2vec", p=2.0, q=0.5), make_app("ppr", termination_probability=0.01)):
    dr = run_device(app, dg, n_samples=V, seed=7); dr.close()
    for c in (1, 3, 6, 12, 24):
        pipe = HostPipeline(chunks=c)
        ms = []
        for it in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); pipe.run_jobs(dg, [(app, V, 7, 0, None, c)]); e.record()
            torch.cuda.synchronize()
            if it: ms.append(s.elapsed_time(e))
        print(app.name, c, round(statistics.median(ms), 2), flush=True)

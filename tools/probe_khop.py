"""Dev probe: C3 k-hop device-only timing per paradigm, 228 batches of 1024
roots as one launch and a single 1024-root batch (ND_TRACE=1 for phases)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
app = make_app("khop")
for par in sys.argv[1:] or ["tp", "sp"]:
    for N in (1024 * 228, 1024):
        ms = []
        for it in range(12):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par)
            e.record()
            torch.cuda.synchronize()
            if it >= 2:
                ms.append(s.elapsed_time(e))
            edges = dr.total_sampled
            dr.close()
        print(par, N, round(statistics.median(ms), 4), edges, flush=True)

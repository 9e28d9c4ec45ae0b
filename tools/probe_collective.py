"""Dev tool: one collective app on the C4 graph (RMAT scale 22, 58.6M
undirected edges) inside cudaProfilerStart/Stop for ncu launch lists."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "clustergcn"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
par = sys.argv[3] if len(sys.argv) > 3 else "tp"
dg = DeviceGraph.rmat(22, n_edges=58_600_000, seed=0, weighted=False, undirected=True)
app = make_app(name)
run_device(app, dg, n_samples=N, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
s.record()
dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par)
e.record()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(json.dumps({"app": name, "N": N, "event_ms": s.elapsed_time(e), "wall_ms": 1e3 * (time.perf_counter() - t0),
                  "recorded": dr.total_recorded, "sampled": dr.total_sampled}))
dr.close()

"""Dev tool: one bench step (node2vec + PPR, SP) inside cudaProfilerStart/Stop
for `ncu --profile-from-start off` launch lists; also prints phase timings."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

par = sys.argv[1] if len(sys.argv) > 1 else "sp"
dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
N = dg.n_vertices
apps = [make_app("node2vec"), make_app("ppr")]
L = _lib.load()
L.nd_set_profiling(1)
for _ in range(2):
    for a in apps:
        run_device(a, dg, n_samples=N, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for a in apps:
    t0 = time.perf_counter()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    dr = run_device(a, dg, n_samples=N, seed=7, paradigm=par)
    e.record()
    torch.cuda.synchronize()
    print(json.dumps({"app": a.name, "event_ms": s.elapsed_time(e), "wall_ms": 1e3 * (time.perf_counter() - t0),
                      "prof_ms": dr.profile_ms, "launches": dr.counters["launches"],
                      "edges": dr.total_sampled}), flush=True)
    dr.close()
torch.cuda.cudart().cudaProfilerStop()

"""Dev probe: time device walks (TP vs SP) on an RMAT graph; prints JSON lines."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2009_06693_b200 import make_app, _lib  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
n_edges = int(sys.argv[2]) if len(sys.argv) > 2 else 68_993_773
t0 = time.perf_counter()
dg = DeviceGraph.rmat(scale, n_edges=n_edges, seed=0, weighted=True)
torch.cuda.synchronize()
print(json.dumps({"graph_build_s": time.perf_counter() - t0, "V": dg.n_vertices, "E": dg.n_edges,
                  "bytes": dg.bytes}), flush=True)
N = dg.n_vertices
for app_name in ("deepwalk", "node2vec", "ppr"):
    app = make_app(app_name)
    for par in ("tp", "sp"):
        for prof in (0, 1):
            _lib.load().nd_set_profiling(prof)
            dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par)  # warm
            dr.close()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e)
            print(json.dumps({"app": app_name, "paradigm": par, "profile": prof, "ms": ms,
                              "edges": dr.total_sampled, "Gedges_s": dr.total_sampled / ms / 1e6,
                              "steps": dr.n_steps, "counters": dr.counters,
                              "prof_ms": dr.profile_ms,
                              "model_GBs": dr.counters["slot_bytes"] / ms / 1e6}), flush=True)
            dr.close()

"""Does node2vec fit on the C5 graph (RMAT-26, 1,073,741,824 weighted edges)
on one B200?  Builds the graph, runs DeepWalk then node2vec on 2^20 walkers,
and reports the footprint of every lazily built structure (built or left out
for lack of room: then the kernels read the plain CSR), the device time of
each run, and the HBM left.

  python tools/probe_c5_node2vec.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

t0 = time.perf_counter()
dg = DeviceGraph.rmat(26, n_edges=1 << 30, seed=0, weighted=True)
torch.cuda.synchronize()
out = {"graph": "C5 RMAT-26, 1,073,741,824 weighted edges", "build_s": time.perf_counter() - t0,
       "runs": []}
n = 1 << 20
for name, kw in (("deepwalk", {}), ("node2vec", {"p": 2.0, "q": 0.5})):
    app = make_app(name, **kw)
    for it in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dr = run_device(app, dg, n_samples=n, seed=7, paradigm="sp")
        e1.record()
        torch.cuda.synchronize()
        fr, tot = torch.cuda.mem_get_info()
        out["runs"].append({"app": name, "iter": it, "ms": e0.elapsed_time(e1),
                            "edges": dr.total_sampled,
                            "edges_per_s": dr.total_sampled / e0.elapsed_time(e1) * 1e3,
                            "footprint": dg.footprint(), "hbm_free_gb": fr / 1e9,
                            "hbm_total_gb": tot / 1e9})
        dr.close()
print(json.dumps(out, indent=1))

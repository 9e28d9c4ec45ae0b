"""C5 DeepWalk kernel time (2^23 walkers on the 1.07B-edge graph) in a fresh
process, or after other work has allocated and freed device memory first
(argv[1] = "fresh" | "after-c2"): checks whether the placement of the 110 GB
of graph structures (and so the GPU's translation reach over them) depends
on what the process allocated before."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fresh"
L = _lib.load()
if mode == "after-c2":
    g2 = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
    for name in ("node2vec", "ppr"):
        run_device(make_app(name), g2, n_samples=g2.n_vertices, seed=7, paradigm="sp").close()
        run_device(make_app(name), g2, n_samples=g2.n_vertices, seed=7, paradigm="tp").close()
    g2.close()
    torch.cuda.empty_cache()
t0 = time.perf_counter()
dg = DeviceGraph.rmat(26, n_edges=1 << 30, seed=0, weighted=True)
torch.cuda.synchronize()
build = time.perf_counter() - t0
L.nd_set_profiling(1)
ms = []
for it in range(int(os.environ.get('PROBE_ITERS', '4'))):
    dr = run_device(make_app("deepwalk"), dg, n_samples=1 << 23, seed=7, paradigm="sp")
    ms.append(dr.profile_ms[1])
    dr.close()
print(json.dumps({"mode": mode, "build_s": build, "kernel_ms": ms[1:]}))

"""Dev tool: event-timed node2vec / PPR walks on the C2 graph under the
current environment (ND_WALK_MINB, ND_NO_LINES, ND_NO_PACK, ...); prints one JSON line
per app with the median of 5 runs and the run's byte-model counters."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

scale = int(os.environ.get("AB_SCALE", "22"))
dg = DeviceGraph.rmat(scale, n_edges=68_993_773 if scale == 22 else 16 << scale, seed=0, weighted=True)
N = dg.n_vertices
L = _lib.load()
L.nd_set_profiling(1)
tag = {k: v for k, v in os.environ.items() if k.startswith("ND_")}
for name in sys.argv[1:] or ["node2vec", "ppr", "deepwalk"]:
    a = make_app(name)
    ms, kms = [], []
    for it in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dr = run_device(a, dg, n_samples=N, seed=7, paradigm=os.environ.get("AB_PARADIGM", "sp"))
        e.record()
        torch.cuda.synchronize()
        if it:
            ms.append(s.elapsed_time(e))
            kms.append(dr.profile_ms[1])
        edges, c = dr.total_sampled, dict(dr.counters)
        dr.close()
    print(json.dumps({"env": tag, "app": name, "ms": statistics.median(ms), "kernel_ms": statistics.median(kms),
                      "edges": edges, "Gedges_s": edges / statistics.median(ms) / 1e6,
                      "model_GBs": c["slot_bytes"] / statistics.median(kms) / 1e6, "tries": c["n2v_tries"],
                      "rand_sectors": c["rand_sectors"], "Gsect_s": c["rand_sectors"] / statistics.median(kms) / 1e6}),
          flush=True)

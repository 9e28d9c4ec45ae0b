"""Dev probe: run-to-run modes of the C2 walk kernels.  Each app alone, K
back-to-back runs on one stream, event time per run and the address of the
run's largest allocation (the step window), to see whether the slow / fast
mode follows the placement of the run's buffers.

  python tools/probe_bimodal.py [node2vec|ppr|deepwalk] [K]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
name = sys.argv[1] if len(sys.argv) > 1 else "node2vec"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
app = make_app(name)
L = _lib.load()
L.nd_set_profiling(1)
res = []
for it in range(K + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dr = run_device(app, dg, n_samples=dg.n_vertices, seed=7, paradigm="sp")
    e1.record()
    torch.cuda.synchronize()
    ptr, cnt = dr.field_count(_lib.F_FINAL_IDS)
    if it:
        res.append({"ms": round(e0.elapsed_time(e1), 3), "kernel_ms": round(dr.profile_ms[1], 3),
                    "final_ids_ptr": hex(ptr), "mod_2M": (ptr >> 21) & 0xFFF})
    dr.close()
print(json.dumps({"app": name, "runs": res}))

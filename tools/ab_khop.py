"""A/B of the C3 k-hop run (233,472 roots, fanouts 25,10, RMAT-18 114.6M
edges) under the current environment's knobs: SP and TP event-timed medians,
per-step build/sample times, rows checked against SP.  One JSON line.

  ND_FX_HUB=1 python tools/ab_khop.py
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import profiling, run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
app = make_app("khop", fanouts=[25, 10])
N = 1024 * 228
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("ND_")}}
ref = None
for par in ("sp", "tp"):
    for _ in range(3):
        run_device(app, dg, n_samples=N, seed=7, paradigm=par).close()
    ms = []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par, sync=False)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        if ref is None:
            ref = dr.view(_lib.F_FINAL_IDS32).clone()
        else:
            out.setdefault("rows_equal", True)
            out["rows_equal"] &= bool(torch.equal(ref, dr.view(_lib.F_FINAL_IDS32)))
        dr.close()
    with profiling():
        dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par)
    out[par] = {"ms_median": statistics.median(ms), "ms_min": min(ms), "steps": dr.step_ms,
                "compact_ms": dr.profile_ms[2]}
    dr.close()
out["tp_vs_sp"] = out["tp"]["ms_median"] / out["sp"]["ms_median"]
print(json.dumps(out))

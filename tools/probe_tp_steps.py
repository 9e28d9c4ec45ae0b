"""Where a C2 TP walk spends its time: per-step (build, sample) event times of
the TP step engine (profiling on), the step counts, and the wall time of the
whole run, per app; the SP time beside it.  Lists the first steps, every 8th
step and the totals; steps past the hub engine's last step ran in the
walker-major tail (recorded as one entry per window)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
L = _lib.load()
for name in sys.argv[1:] or ["ppr", "node2vec"]:
    app = make_app(name)
    for paradigm in ("sp", "tp", "tp"):
        L.nd_set_profiling(1 if paradigm == "tp" else 0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        dr = run_device(app, dg, n_samples=dg.n_vertices, seed=7, paradigm=paradigm)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        st = dr.step_ms
        out = {"app": name, "paradigm": paradigm, "ms": round(ms, 3), "steps": dr.n_steps,
               "recorded_steps": len(st), "profile_ms": [round(x, 3) for x in dr.profile_ms]}
        if st:
            out["build_ms"] = round(sum(b for b, _ in st), 3)
            out["sample_ms"] = round(sum(x for _, x in st), 3)
            out["per_step"] = [(i, round(b, 3), round(x, 3)) for i, (b, x) in enumerate(st)
                               if i < 6 or i % 8 == 0 or i == len(st) - 1]
        print(json.dumps(out), flush=True)
        dr.close()
L.nd_set_profiling(0)

"""C3 k-hop (233,472 roots) as one run vs k concurrent runs over contiguous
sample-id blocks (engine.run_device_concurrent: one stream and host thread
per block; the keyed RNG makes the rows identical), SP and TP, event-timed
medians.  One JSON line per (paradigm, k)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device_concurrent  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.sharding import worker_ranges  # noqa: E402

dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
app = make_app("khop", fanouts=[25, 10])
N = 1024 * 228
cur = torch.cuda.current_stream()
for par in ("sp", "tp"):
    ref = None
    for k in (1, 2, 3, 4):
        jobs = [dict(app=app, n_samples=b - a, sample_lo=a, seed=7) for a, b in worker_ranges(N, k)]
        ms = []
        ok = True
        for it in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            runs = run_device_concurrent(jobs, dg, paradigm=par)
            e1.record(cur)
            torch.cuda.synchronize()
            if it >= 3:
                ms.append(e0.elapsed_time(e1))
            ids = torch.cat([r.view(_lib.F_FINAL_IDS32) for r in runs])
            if ref is None:
                ref = ids.clone()
            ok &= bool(torch.equal(ids, ref))
            for r in runs:
                r.close()
        print(json.dumps({"paradigm": par, "blocks": k, "ms_median": statistics.median(ms),
                          "ms_min": min(ms), "rows_equal": ok}), flush=True)

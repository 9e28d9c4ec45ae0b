"""Dev probe: C5 DeepWalk (RMAT-26, 1.07B weighted edges, 2^23 walkers, one
GPU) alone under different persistent-grid sizes (ND_WALK_GRID, CTAs per SM,
read per run) and occupancy builds (ND_WALK_MINB); event-timed kernel time
per run, interleaved so box drift hits every variant alike.

  python tools/probe_c5_walk.py "0=4" "0=3" "0=2" ...
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(26, n_edges=1 << 30, seed=0, weighted=True)
app = make_app("deepwalk")
L = _lib.load()
L.nd_set_profiling(1)
variants = sys.argv[1:] or ["0=4", "0=2"]
res = {v: [] for v in variants}
run_device(app, dg, n_samples=1 << 23, seed=7, paradigm="sp").close()  # builds the indexes
for rep in range(int(os.environ.get("REPS", "4"))):
    for v in variants:
        minb, _, grid = v.partition("/")  # "4/0=2": MINB 4, 2 CTAs per SM
        if grid:
            os.environ["ND_WALK_MINB"] = minb
        else:
            grid = minb
            os.environ.pop("ND_WALK_MINB", None)
        os.environ["ND_WALK_GRID"] = grid
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dr = run_device(app, dg, n_samples=1 << 23, seed=7, paradigm="sp")
        e1.record()
        torch.cuda.synchronize()
        ptr, _ = dr.field_count(_lib.F_FINAL_IDS)
        res[v].append((round(e0.elapsed_time(e1), 2), round(dr.profile_ms[1], 2), hex(ptr)[-9:]))
        dr.close()
        if os.environ.get("TRIM"):  # every run from an emptied allocation pool
            torch.cuda.synchronize()
            L.nd_pool_trim(0)
print(json.dumps({"deepwalk_c5 (run ms, kernel ms)": res}))

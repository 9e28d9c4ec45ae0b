"""Out-of-core shuttling at C2 scale: DeepWalk (4,194,304 walkers x 100),
PPR (4,194,304 walkers, term 0.01), k-hop (25,10) x 233,472 roots and
node2vec (4,194,304 walkers, read in place from host memory: zero copy) on the C2 RMAT graph held in host memory with a
device budget that cuts it into ~4 partitions, against the in-core runs of
the same jobs (rows compared, times event-based, shuttled bytes reported).

  python tools/probe_ooc.py [parts]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.outofcore import ShuttledGraph  # noqa: E402

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
hg = dg.to_host()
budget = (dg.n_vertices + 1) * 8 + 2 * 12 * (dg.n_edges // parts + 1)
t0 = time.perf_counter()
sg = ShuttledGraph.from_graph(hg, device_budget_bytes=budget)
reg_s = time.perf_counter() - t0
out = {"graph": "C2 RMAT-22, 68,993,773 weighted edges", "budget_bytes": budget,
       "register_s": reg_s, **sg.info()}


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dr = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), dr


for name, kw, n in (("deepwalk", {}, dg.n_vertices), ("ppr", {}, dg.n_vertices),
                    ("khop", {"fanouts": [25, 10]}, 1024 * 228),
                    ("node2vec", {"p": 2.0, "q": 0.5}, dg.n_vertices)):  # zero copy
    app = make_app(name, **kw)
    res = {}
    rows = {}
    for where, g in (("in_core", dg), ("out_of_core", sg)):
        run_device(app, g, n_samples=min(n, 4096), seed=7).close()  # warm-up (indexes, pools)
        b0 = sg.info()["bytes_shuttled"]
        ms, dr = timed(lambda: run_device(app, g, n_samples=n, seed=7, paradigm="sp"))
        rows[where] = (dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS))
        res[where] = {"ms": ms, "edges": dr.total_sampled, "edges_per_s": dr.total_sampled / ms * 1e3}
        if where == "out_of_core":
            res[where]["bytes_shuttled"] = sg.info()["bytes_shuttled"] - b0
            res[where]["rounds_or_steps"] = dr.counters["steps"]
            res[where]["pcie_gbs"] = res[where]["bytes_shuttled"] / ms / 1e6
        dr.close()
    res["rows_equal"] = bool(np.array_equal(rows["in_core"][0], rows["out_of_core"][0])
                             and np.array_equal(rows["in_core"][1], rows["out_of_core"][1]))
    out[name] = res
print(json.dumps(out, indent=1))

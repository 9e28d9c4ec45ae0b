"""TP vs SP walks as the number of walkers per vertex grows (the paper's TP
pays when a transit's members share its adjacency): DeepWalk / node2vec / PPR
on RMAT-18 (262,144 V, 4.3M weighted edges) with N = k * V walkers, k in
{1, 4, 16, 32}; event-timed runs, rows compared, and the share of walker-steps
the TP engine sampled from staged rows (tp_staged)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

scale = int(os.environ.get("DENSITY_SCALE", "18"))
dg = DeviceGraph.rmat(scale, n_edges=int(68_993_773 / (1 << 22) * (1 << scale)), seed=0, weighted=True)
V = dg.n_vertices
apps = sys.argv[1:] or ["deepwalk", "node2vec", "ppr"]
for name in apps:
    app = make_app(name)
    for k in (1, 4, 16, 32):
        N = k * V
        res = {"app": name, "walkers_per_vertex": k, "N": N}
        ids = {}
        for par in ("sp", "tp"):
            run_device(app, dg, n_samples=N, seed=7, paradigm=par).close()
            ms = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dr = run_device(app, dg, n_samples=N, seed=7, paradigm=par, sync=False)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
                c = dr.counters
                ids[par] = dr.view(_lib.F_FINAL_IDS32).sum().item()
                edges = dr.total_sampled
                dr.close()
            res[par] = {"ms": statistics.median(ms), "edges_per_s": edges / statistics.median(ms) * 1e3}
            if par == "tp":
                res["tp_staged_share"] = c["tp_staged"] / max(1, c["tp_staged"] + c["tp_inplace"])
        res["tp_over_sp"] = res["tp"]["ms"] / res["sp"]["ms"]
        res["rows_checksum_equal"] = ids["sp"] == ids["tp"]
        print(json.dumps(res), flush=True)

"""Small end-to-end runs of every engine path, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2009_06693_b200 import kernels as K, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.schedule import transit_schedule  # noqa: E402

dg = DeviceGraph.rmat(10, 16, seed=2, weighted=True)
du = DeviceGraph.rmat(10, 8, seed=3, undirected=True, weighted=False)
runs = [("deepwalk", {}, dg), ("ppr", {}, dg), ("node2vec", {}, dg), ("multirw", {"roots_per_sample": 8}, dg),
        ("khop", {}, du), ("layer", {"max_size": 200, "step_size": 50}, du), ("fastgcn", {}, du),
        ("ladies", {"distribution": "degree_sq"}, du), ("mvs", {}, du),
        ("clustergcn", {"clusters_per_sample": 3, "num_clusters": 10}, du)]
for name, kw, g in runs:
    for par in ("sp", "tp"):
        app = make_app(name, **kw)
        if name == "khop" and par == "tp":
            app.unique = lambda s: s == 0
        dr = run_device(app, g, n_samples=300, seed=5, paradigm=par)
        dr.to_output()
        dr.close()
h = dg.to_host()
n = 5000
rng = np.random.default_rng(1)
out = np.empty(n, dtype=np.int64)
for code, prm in ((0, []), (1, [0.1]), (2, [2.0, 0.5, 0.0]), (3, []), (4, [])):
    K.individual_batch(code, prm, h.row_offsets, h.col_indices, h.weights, h.per_vertex_weight_prefix,
                       h.per_vertex_max_weight, rng.integers(0, h.n_vertices, n), rng.integers(-1, h.n_vertices, n),
                       rng.integers(0, 1000, n), rng.integers(0, 5, n), rng.integers(0, 5, n), 7, 1, out)
transit_schedule(rng.integers(0, 50, 2000), 3)
print("sanitize smoke ok")

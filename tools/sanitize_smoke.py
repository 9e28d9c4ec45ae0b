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
import os  # noqa: E402
for name, kw, g in runs:
    for par in ("sp", "tp"):
        if par == "tp" and name in ("ppr", "node2vec", "deepwalk"):
            # TP walks: all steps in the class kernels, then a mid-run hand-off to the tail
            # (and with the staged tiers off: k_tw_multi, 3 and 4 steps per launch)
            for tail, stage, multi in (("0", None, None), ("100", None, None), ("0", "0", "3"),
                                       ("0", "0", "4")):
                os.environ["ND_TP_TAIL"] = tail
                for k, v in (("ND_TW_STAGE", stage), ("ND_TW_MULTI", multi)):
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
                dr = run_device(make_app(name, **kw), g, n_samples=300, seed=5, paradigm=par)
                dr.to_output()
                dr.close()
            for k in ("ND_TP_TAIL", "ND_TW_STAGE", "ND_TW_MULTI"):
                os.environ.pop(k, None)
        for uniq in ((False, True) if name == "khop" else (False,)):
            app = make_app(name, **kw)
            if uniq:  # the step-loop engine (unique steps); otherwise the fixed layout
                app.unique = lambda s: s == 0
            dr = run_device(app, g, n_samples=300, seed=5, paradigm=par)
            dr.to_output()
            dr.final_samples()
            dr.close()
# edge-list ingestion on device (one non-ASCII line goes through the host)
import os, tempfile  # noqa: E402
with tempfile.TemporaryDirectory() as td:
    path = os.path.join(td, "e.txt")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("# c\n0 1 2.5\n1 2\r\n2 0 1e-3\n\u0663 4 0.5\n4 0 7\r5 4\n")
    g2 = DeviceGraph.from_edge_list(path, weighted=True, undirected=True)
    dr = run_device(make_app("ppr"), g2, n_samples=50, seed=1, paradigm="sp")
    dr.close()
    g2.close()
from paper_2009_06693_b200 import _lib  # noqa: E402
import ctypes as C  # noqa: E402
c = C.c_double()
_lib.load().nd_gather_ceiling(64 << 20, 1, 4, C.byref(c), None)
h = dg.to_host()
n = 5000
rng = np.random.default_rng(1)
out = np.empty(n, dtype=np.int64)
for code, prm in ((0, []), (1, [0.1]), (2, [2.0, 0.5, 0.0]), (3, []), (4, [])):
    K.individual_batch(code, prm, h.row_offsets, h.col_indices, h.weights, h.per_vertex_weight_prefix,
                       h.per_vertex_max_weight, rng.integers(0, h.n_vertices, n), rng.integers(-1, h.n_vertices, n),
                       rng.integers(0, 1000, n), rng.integers(0, 5, n), rng.integers(0, 5, n), 7, 1, out)
transit_schedule(rng.integers(0, 50, 2000), 3)
# round 2: step timing (events per step), the k-hop TP hub tiers on a denser
# graph (warp and thread-block tiers), out-of-core shuttling, ShardedJob
from paper_2009_06693_b200.engine import profiling  # noqa: E402
from paper_2009_06693_b200.multigpu import ShardedJob  # noqa: E402
from paper_2009_06693_b200.outofcore import ShuttledGraph  # noqa: E402
dd = DeviceGraph.rmat(10, 64, seed=4, undirected=True, weighted=False)
with profiling():
    for par in ("sp", "tp"):
        dr = run_device(make_app("khop", fanouts=[25, 10]), dd, n_samples=2000, seed=5, paradigm=par)
        dr.to_output()
        dr.close()
        dr = run_device(make_app("fastgcn"), du, n_samples=64, seed=5, paradigm=par)
        dr.close()
hg = dg.to_host()
sg = ShuttledGraph.from_graph(hg, device_budget_bytes=(hg.n_vertices + 1) * 8 + 2 * 12 * (hg.n_edges // 4 + 64))
for name, kw in (("deepwalk", {"walk_length": 20}), ("khop", {"fanouts": [5, 3]}),
                 ("ppr", {"termination_probability": 0.05}), ("node2vec", {"walk_length": 10}),
                 ("fastgcn", {"batch_size": 8, "step_size": 8, "steps": 2})):
    dr = run_device(make_app(name, **kw), sg, n_samples=300, seed=5)  # shuttled / zero copy
    dr.to_output()
    dr.close()
sg.close()
from paper_2009_06693_b200.minibatch import KhopBatchSampler  # noqa: E402
import torch  # noqa: E402
smp = KhopBatchSampler(du, [5, 3], 256)
for b in range(3):
    smp.sample(torch.randint(0, du.n_vertices, (256,), device="cuda", dtype=torch.int64),
               sample_lo=b * 256, seed=5)
torch.cuda.synchronize()
smp.close()
job = ShardedJob(dg, [(make_app("deepwalk"), 500, 5, 3), (make_app("khop"), 200, 5)], to_host=True)
job.run(order=[1, 0])
# text rows printed on the device (nd_format_rows), both layouts, with gpu_share
from paper_2009_06693_b200 import output as OUT  # noqa: E402
from paper_2009_06693_b200.engine import gpu_share  # noqa: E402
OUT.DEVICE_FORMAT_MIN_IDS = 0
for name in ("node2vec", "khop"):
    with gpu_share(2):
        o = run_device(make_app(name), dg, n_samples=300, seed=5).to_output()
    for layout in (OUT.LAYOUT_FINAL, OUT.LAYOUT_PER_STEP):
        OUT.render_bytes(o, layout)
print("sanitize smoke ok")

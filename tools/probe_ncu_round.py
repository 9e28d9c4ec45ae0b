"""ncu workloads of the round's profile capture (tools/ncu_round.sh): one
warm-up run, then the measured run(s) inside cudaProfilerStart/Stop so
`ncu --profile-from-start off` sees exactly one job.

  walk_sp     C2 node2vec + PPR, walker-major SP kernel (the bench's kernel)
  walk_tp     C2 node2vec + PPR through tp_run's hub engine
  khop        C3 k-hop (25,10), 233,472 roots, SP then TP
  dedup       C3 k-hop (25,10) with unique() steps, 16,384 roots (segmented sort + distinct scan)
  collective  C4 FastGCN (4,096 samples) and ClusterGCN (8 samples), TP
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

which = sys.argv[1]
jobs = []
if which in ("walk_sp", "walk_tp"):
    g = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
    par = which[-2:]
    jobs = [(make_app("node2vec", p=2.0, q=0.5), g.n_vertices, par),
            (make_app("ppr", termination_probability=0.01), g.n_vertices, par)]
elif which in ("khop", "dedup"):
    g = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
    app = make_app("khop", fanouts=[25, 10])
    if which == "dedup":
        app.unique = lambda step: True
        jobs = [(app, 1 << 14, "tp")]
    else:
        jobs = [(app, 1024 * 228, "sp"), (app, 1024 * 228, "tp")]
elif which == "collective":
    g = DeviceGraph.rmat(22, n_edges=58_600_000, seed=0, undirected=True, weighted=False)
    jobs = [(make_app("fastgcn"), 4096, "tp"), (make_app("clustergcn"), 8, "tp")]
else:
    raise SystemExit(f"unknown workload {which}")
for app, n, par in jobs:
    run_device(app, g, n_samples=n, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for app, n, par in jobs:
    run_device(app, g, n_samples=n, seed=7, paradigm=par).close()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("probe ok", which, flush=True)

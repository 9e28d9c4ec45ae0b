import os, sys, statistics, json
sys.path.insert(0, "/root/repo" if os.path.exists("/root/repo") else ".")
import torch
from paper_2009_06693_b200 import _lib, make_app
from paper_2009_06693_b200.engine import run_device, run_device_concurrent
from paper_2009_06693_b200.graph import DeviceGraph
L = _lib.load()
def c3(tag):
    dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
    app = make_app("khop", fanouts=[25, 10])
    out = {"tag": tag}
    for par in ("sp", "tp"):
        for _ in range(3): run_device(app, dg, n_samples=233472, seed=7, paradigm=par).close()
        ms = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); dr = run_device(app, dg, n_samples=233472, seed=7, paradigm=par, sync=False); e1.record()
            torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1)); dr.close()
        out[par] = statistics.median(ms)
    dg.close()
    print(json.dumps(out), flush=True)
c3("fresh")
g2 = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
apps = [make_app("node2vec"), make_app("ppr")]
for par in ("sp", "tp", "sp"):
    for r in run_device_concurrent([dict(app=a, n_samples=g2.n_vertices, seed=7) for a in apps], g2, paradigm=par):
        r.close()
g2.close(); torch.cuda.empty_cache()
c3("after-c2")
L.nd_pool_trim(0)
c3("after-c2-trim")

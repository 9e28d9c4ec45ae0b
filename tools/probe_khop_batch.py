import sys, time, statistics, torch
sys.path.insert(0, "/root/repo")
from paper_2009_06693_b200 import make_app
from paper_2009_06693_b200.engine import run_device
from paper_2009_06693_b200.graph import DeviceGraph
dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
app = make_app("khop")
for it in range(30):
    t0 = time.perf_counter()
    dr = run_device(app, dg, n_samples=1024, sample_lo=1024 * it, seed=7, paradigm="sp")
    t1 = time.perf_counter()
    dr.close()
    if it == 29: print("host run_device ms", (t1 - t0) * 1e3)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for it in range(200):
    dr = run_device(app, dg, n_samples=1024, sample_lo=1024 * it, seed=7, paradigm="sp"); dr.close()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)

"""Dev probe: C2 node2vec final rows printed as text on the device
(output.render_bytes -> nd_format_rows) against the Python writer on 1/64 of the rows."""
import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2009_06693_b200 import make_app, output as O
from paper_2009_06693_b200.engine import run_device
from paper_2009_06693_b200.graph import DeviceGraph
dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
dr = run_device(make_app("node2vec"), dg, n_samples=dg.n_vertices, seed=7, paradigm="sp")
out = dr.to_output(); dr.close()
off, ids = out.final_csr()
print("rows", len(off) - 1, "ids", len(ids), flush=True)
for it in range(2):
    t0 = time.perf_counter(); b = O.render_bytes(out, O.LAYOUT_FINAL); t1 = time.perf_counter()
    print("device render_bytes s", round(t1 - t0, 3), "bytes", len(b), flush=True)
t0 = time.perf_counter(); O.emit(out, O.LAYOUT_FINAL, "/tmp/c2_rows.txt"); t1 = time.perf_counter()
print("device emit to /tmp s", round(t1 - t0, 3), flush=True)
# python writer on a 1/64 slice, extrapolated
k = (len(off) - 1) // 64
t0 = time.perf_counter(); lines = []; O._fmt_rows(out.sample_ids[:k], off[:k + 1], ids, lines); t1 = time.perf_counter()
print("python writer s (1/64 of rows)", round(t1 - t0, 3), "-> full est", round((t1 - t0) * 64, 1), flush=True)

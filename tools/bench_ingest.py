"""Ingestion benchmark: edge-list text -> device CSR.

Generates a weighted edge list with tools/gen_edgelist (C2-sized by default:
69M lines, RMAT scale-22 id range), then times
  * device: DeviceGraph.from_edge_list (file read + H2D + parse + id
    compaction + CSR build), median of 3, and the same from bytes already in
    host memory (parse + build only);
  * CPU: the host restatement of the reference parser (load_edge_list, same
    rules as trawl.graph.load_edge_list) on a bounded prefix of the file.
Prints one JSON object.

    python tools/bench_ingest.py [n_lines] [cpu_lines]
"""
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2009_06693_b200.graph import DeviceGraph, load_edge_list  # noqa: E402

n_lines = int(sys.argv[1]) if len(sys.argv) > 1 else 69_000_000
cpu_lines = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
gen = os.path.join(REPO, "tools", "gen_edgelist")
if not os.path.exists(gen):
    subprocess.check_call(["gcc", "-O2", "-o", gen, gen + ".c"])
td = tempfile.mkdtemp()
path = os.path.join(td, "edges.txt")
with open(path, "wb") as fh:
    subprocess.check_call([gen, "22", str(n_lines)], stdout=fh)
size = os.path.getsize(path)

dev = []
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg = DeviceGraph.from_edge_list(path, weighted=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if it:
        dev.append(dt)
    V, E = dg.n_vertices, dg.n_edges
    dg.close()

cpu_path = os.path.join(td, "prefix.txt")
with open(path, "rb") as src, open(cpu_path, "wb") as dst:
    for _ in range(cpu_lines):
        dst.write(src.readline())
t0 = time.perf_counter()
g = load_edge_list(cpu_path, weighted=True)
cpu_s = time.perf_counter() - t0

ms = statistics.median(dev) * 1e3
print(json.dumps({
    "what": "edge-list text -> CSR (load_edge_list semantics, weighted, 3 fields per line)",
    "file_bytes": size, "lines": n_lines, "n_vertices": V, "n_edges": E,
    "device_ms": ms, "device_lines_per_s": n_lines / (ms / 1e3), "device_GB_per_s": size / (ms / 1e3) / 1e9,
    "device_note": "file read + H2D + parse + id compaction + CSR build, median of 3",
    "cpu_lines": cpu_lines, "cpu_s": cpu_s, "cpu_lines_per_s": cpu_lines / cpu_s,
    "cpu_kind": "port: host restatement of trawl.graph.load_edge_list (1 core)",
    "speedup": (n_lines / (ms / 1e3)) / (cpu_lines / cpu_s),
}))

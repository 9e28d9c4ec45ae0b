"""Sweep of the BASELINE.json configs beyond the headline (C1, C3, C4, C5-lite):
device throughput (SP and TP where both exist), the CPU oracle on a bounded
sample of the same job, and parity of that sample.  Writes one JSON object
per config to stdout (collected into profiles/r01_configs.json).

    python -m tests.config_sweep [C1 C3 C4 C5]   (lives under tests/: it runs the C oracle as the CPU baseline and parity checker)
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (CPU baseline + parity only)
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.synth import powerlaw_graph  # noqa: E402

CORES = len(os.sched_getaffinity(0))


def timed(fn, reps=3):
    fn()  # warm
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = fn()
        e.record()
        torch.cuda.synchronize()
        out.append((s.elapsed_time(e), r))
    ms = sorted(x[0] for x in out)[len(out) // 2]
    return ms, out[-1][1]


def og_of(dg):
    h = dg.to_host()
    return O.OGraph(h.n_vertices, h.row_offsets, h.col_indices, h.weights,
                    h.per_vertex_weight_prefix, h.per_vertex_max_weight, None)


class _Lazy:
    """Device run kept resident; host copies only when asked (outside timing)."""

    def __init__(self, dr):
        self.dr = dr

    def __getitem__(self, k):
        if k == 0:
            return self.dr.total_sampled
        if k == 1:
            return self.dr.total_recorded
        if k == 2:
            return self.dr.host(_lib.F_FINAL_OFF)
        return self.dr.host(_lib.F_FINAL_IDS)


def dev_rows(app, dg, n, seed, par, lo=0):
    """Device-only run: outputs stay in HBM (the timed region ends there)."""
    return _Lazy(run_device(app, dg, n_samples=n, sample_lo=lo, seed=seed, paradigm=par))


def c1():
    g = powerlaw_graph(56944, attach=7, weighted=True, seed=0)
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    app = make_app("deepwalk")
    N, seed = g.n_vertices, 7
    res = {"config": "C1 PPI-shaped DeepWalk: powerlaw(56944, attach 7, weighted, seed 0), "
                     "len 100, N=V", "V": g.n_vertices, "E": len(g.col_indices),
           "note": "whole graph (~20 MB) is L2-resident: HBM % not binding"}
    for par in ("sp", "tp"):
        ms, r = timed(lambda: dev_rows(app, dg, N, seed, par))
        res[par] = {"ms": ms, "edges": r[0], "edges_per_s": r[0] / ms * 1e3}
    og = og_of(dg)
    roots = O.uniform_roots(og.n_vertices, 1, seed, 0, N)
    t0 = time.perf_counter()
    ref = O.run_chain(og, 0, [], roots, seed, 100, paradigm="sp", n_threads=CORES)
    dt = time.perf_counter() - t0
    edges = int((ref["chain_vals"] >= 0).sum())
    res["cpu"] = {"s": dt, "edges_per_s": edges / dt, "cores": CORES, "kind": "port", "sample": "full job"}
    r = dev_rows(app, dg, N, seed, "sp")
    off, ids = r[2], r[3]
    cl = ref["chain_len"]
    st = np.concatenate([[0], np.cumsum(cl)])
    exp = np.concatenate([np.concatenate([roots[i], ref["chain_vals"][st[i]:st[i + 1]][ref["chain_vals"][st[i]:st[i + 1]] >= 0]]) for i in range(N)])
    res["parity"] = bool(np.array_equal(ids, exp))
    return res


def c3():
    dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
    app = make_app("khop", fanouts=[25, 10])
    B, seed = 228, 7
    N = 1024 * B
    res = {"config": "C3 Reddit-shaped k-hop (25,10): RMAT scale 18, 57.3M undirected edges "
                     "(114.6M directed), unit weights; 228 batches of 1024 roots as one launch",
           "V": dg.n_vertices, "E": dg.n_edges}
    for par in ("sp", "tp"):
        ms, r = timed(lambda: dev_rows(app, dg, N, seed, par))
        ms1, r1 = timed(lambda: dev_rows(app, dg, 1024, seed, par))
        res[par] = {"ms": ms, "edges": r[0], "edges_per_s": r[0] / ms * 1e3,
                    "single_batch_ms": ms1, "single_batch_edges": r1[0]}
    og = og_of(dg)
    ncpu = 1 << 14
    roots = list(O.uniform_roots(og.n_vertices, 1, seed, 0, ncpu))
    t0 = time.perf_counter()
    ref = O.run_individual(og, 3, [], [25, 10], roots, seed, 2, paradigm="sp")
    dt = time.perf_counter() - t0
    edges = int((ref["vals"] >= 0).sum())
    res["cpu"] = {"s": dt, "edges_per_s": edges / dt, "cores": 1, "kind": "port",
                  "sample": f"k-hop roots [0, {ncpu})"}
    dr = run_device(app, dg, n_samples=ncpu, seed=seed, paradigm="tp")
    out = dr.to_output()
    res["parity"] = bool(np.array_equal(out.step_vals, ref["vals"]))
    dr.close()
    return res


def c4():
    dg = DeviceGraph.rmat(22, n_edges=58_600_000, seed=0, undirected=True, weighted=False)
    res = {"config": "C4 Orkut-shaped collective: RMAT scale 22, 58.6M undirected (117.2M directed), "
                     "unit weights", "V": dg.n_vertices, "E": dg.n_edges, "apps": {}}
    og = og_of(dg)
    seed = 7
    for name, kw, N, ncpu in (("fastgcn", {}, 4096, 256), ("ladies", {"distribution": "degree_sq"}, 4096, 256),
                              ("mvs", {}, 4096, 4096), ("clustergcn", {}, 8, 1)):
        app = make_app(name, **kw)
        ms, r = timed(lambda: dev_rows(app, dg, N, seed, "tp"), reps=3)
        ent = {"N": N, "ms": ms, "sampled": r[0], "recorded": r[1],
               "edges_per_s": (r[0] + r[1]) / ms * 1e3, "unit": "sampled + recorded edges/s"}
        from tests.helpers import app_spec  # noqa: E402
        sp = app_spec(name, kw)
        if name == "clustergcn":
            roots = [O.cluster_roots(og.n_vertices, 20, 100, seed, i) for i in range(ncpu)]
        else:
            roots = list(O.uniform_roots(og.n_vertices, sp["R"], seed, 0, ncpu))
        t0 = time.perf_counter()
        ref = O.run_collective(og, sp["kind"], sp["m"], roots, seed, sp["steps"],
                               distribution=sp.get("distribution", 0))
        dt = time.perf_counter() - t0
        e = int((ref["vals"] >= 0).sum()) + len(ref["rec_t"])
        ent["cpu"] = {"s": dt, "edges_per_s": e / dt, "cores": 1, "kind": "port",
                      "sample": f"sample ids [0, {ncpu})"}
        dr = run_device(app, dg, n_samples=ncpu, seed=seed)
        out = dr.to_output()
        ent["parity"] = bool(np.array_equal(out.step_vals, ref["vals"]) and
                             np.array_equal(out.rec_t, ref["rec_t"]) and
                             np.array_equal(out.rec_v, ref["rec_v"]))
        dr.close()
        res["apps"][name] = ent
    return res


def c5():
    """1B-edge RMAT (scale 26, 1,073,741,824 weighted directed edges) on one
    GPU: DeepWalk 2^23 walkers x 100 and k-hop 2^20 roots; the per-GPU share of
    the 8-GPU sharded job."""
    t0 = time.perf_counter()
    dg = DeviceGraph.rmat(26, n_edges=1 << 30, seed=0, weighted=True)
    torch.cuda.synchronize()
    res = {"config": "C5 RMAT scale 26, 1,073,741,824 weighted directed edges (one GPU)",
           "V": dg.n_vertices, "E": dg.n_edges, "graph_build_s": time.perf_counter() - t0,
           "graph_bytes": dg.bytes}
    for name, N in (("deepwalk", 1 << 23), ("khop", 1 << 20)):
        app = make_app(name)
        ms, r = timed(lambda: dev_rows(app, dg, N, 7, "sp"), reps=2)
        res[name] = {"N": N, "ms": ms, "edges": r[0], "edges_per_s": r[0] / ms * 1e3}
    return res


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C3", "C4"]
    for w in which:
        out = {"C1": c1, "C3": c3, "C4": c4, "C5": c5}[w]()
        print(json.dumps(out), flush=True)

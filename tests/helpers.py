"""Shared test helpers: golden fixtures and oracle-result adapters."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle import oracle as O
from paper_2009_06693_b200.output import LAYOUT_FINAL, LAYOUT_PER_STEP, SampleSetOutput, render_text

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_cache = {}


def golden(name):
    if name not in _cache:
        path = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            with open(path) as fh:
                _cache[name] = json.load(fh)
        else:
            _cache[name] = dict(np.load(path))
    return _cache[name]


def golden_graph(key) -> O.OGraph:
    g = golden("graphs.npz")
    return O.OGraph(len(g[f"{key}/row_offsets"]) - 1, g[f"{key}/row_offsets"],
                    g[f"{key}/col_indices"], g[f"{key}/weights"], g[f"{key}/prefix"],
                    g[f"{key}/max_w"], np.arange(len(g[f"{key}/row_offsets"]) - 1))


def sha16(text):
    return hashlib.sha256(text.encode()).hexdigest()[:16]


APP_CODES = {"deepwalk": 0, "ppr": 1, "node2vec": 2, "khop": 3, "multirw": 4}
COLLECTIVE_KINDS = {"layer": 0, "fastgcn": 1, "ladies": 1, "mvs": 2, "clustergcn": 3}


def unique_mask(params, n=64):
    """The golden cases' unique() spec: "all" or a list of unique steps."""
    u = params.get("unique")
    if u is None:
        return None
    if u == "all":
        return [1] * n
    return [1 if s in u else 0 for s in range(n)]


def app_spec(app, params):
    """Reference defaults (apps.py:37-80) merged with the overrides."""
    p = {k: v for k, v in params.items() if k != "unique"}
    if app == "deepwalk":
        return dict(code=0, kparams=[], steps=p.get("walk_length", 100), R=1)
    if app == "ppr":
        return dict(code=1, kparams=[p.get("termination_probability", 0.01)], steps=None, R=1)
    if app == "node2vec":
        conv = p.get("factor_convention", "reciprocal")
        return dict(code=2, kparams=[p.get("p", 2.0), p.get("q", 0.5), 0.0 if conv == "reciprocal" else 1.0],
                    steps=p.get("walk_length", 100), R=1)
    if app == "multirw":
        return dict(code=4, kparams=[], steps=p.get("walk_length", 100), R=p.get("roots_per_sample", 100))
    if app == "khop":
        f = p.get("fanouts", [25, 10])
        return dict(code=3, kparams=[], steps=len(f), fanouts=f, R=1)
    if app in ("fastgcn", "ladies"):
        return dict(kind=1, m=p.get("step_size", 64), steps=p.get("steps", 5), R=p.get("batch_size", 64),
                    distribution=1 if p.get("distribution", "uniform") == "degree_sq" else 0)
    if app == "mvs":
        return dict(kind=2, m=p.get("step_size", 64), steps=1, R=p.get("batch_size", 64))
    if app == "layer":
        return dict(kind=0, m=p.get("step_size", 1000), steps=None, R=1, max_size=p.get("max_size", 2000))
    if app == "clustergcn":
        return dict(kind=3, m=1, steps=1, cps=p.get("clusters_per_sample", 20), nc=p.get("num_clusters", 100))
    raise ValueError(app)


def oracle_run(meta, g: O.OGraph, paradigm="tp", n_threads=1, step_cap=10_000):
    """Run one golden case through the C oracle; returns SampleSetOutput."""
    app, n, seed = meta["app"], meta["n_samples"], meta["seed"]
    sp = app_spec(app, meta["params"])
    ids = np.arange(n, dtype=np.int64)
    if app == "clustergcn":
        roots = [O.cluster_roots(g.n_vertices, sp["cps"], sp["nc"], seed, i) for i in range(n)]
    else:
        roots = list(O.uniform_roots(g.n_vertices, sp["R"], seed, 0, n))
    um = unique_mask(meta["params"])
    if "kind" in sp:
        r = O.run_collective(g, sp["kind"], sp["m"], roots, seed, sp["steps"],
                             max_size=sp.get("max_size", 0), distribution=sp.get("distribution", 0),
                             unique=um, step_cap=step_cap)
        roff = np.concatenate([[0], np.cumsum([len(x) for x in roots])])
        out = SampleSetOutput(ids, roff, np.concatenate(roots), r["n_steps"], stats=r["stats"],
                              step_counts=r["step_counts"], step_vals=r["vals"],
                              rec_counts=r["rec_counts"], rec_t=r["rec_t"], rec_v=r["rec_v"])
        return out
    if app == "khop":
        r = O.run_individual(g, 3, [], sp["fanouts"], roots, seed, sp["steps"], paradigm=paradigm,
                             unique=um, step_cap=step_cap)
        roff = np.concatenate([[0], np.cumsum([len(x) for x in r["roots"]])])
        return SampleSetOutput(ids, roff, np.concatenate(r["roots"]), r["n_steps"], stats=r["stats"],
                               step_counts=r["step_counts"], step_vals=r["vals"])
    r = O.run_chain(g, sp["code"], sp["kparams"], np.asarray(roots), seed, sp["steps"],
                    paradigm=paradigm, n_threads=n_threads, step_cap=step_cap)
    R = r["roots"].shape[1]
    return SampleSetOutput(ids, np.arange(n + 1) * R, r["roots"].ravel(), r["n_steps"], stats=r["stats"],
                           chain_off=np.concatenate([[0], np.cumsum(r["chain_len"])]),
                           chain_vals=r["chain_vals"])


def texts(out):
    return render_text(out, LAYOUT_FINAL), render_text(out, LAYOUT_PER_STEP)


def recorded_equal(out, rstore, pre):
    if out.rec_t is None or rstore[f"{pre}/rec_cnt"].shape[0] == 0:
        return (out.rec_t is None or len(out.rec_t) == 0) and len(rstore[f"{pre}/rec_t"]) == 0
    return (np.array_equal(np.asarray(out.rec_counts), rstore[f"{pre}/rec_cnt"])
            and np.array_equal(out.rec_t, rstore[f"{pre}/rec_t"])
            and np.array_equal(out.rec_v, rstore[f"{pre}/rec_v"]))


def build_app(meta):
    """make_app with the golden case's overrides, incl. the unique() spec."""
    from paper_2009_06693_b200 import make_app
    kw = {k: v for k, v in meta["params"].items() if k != "unique"}
    app = make_app(meta["app"], **kw)
    u = meta["params"].get("unique")
    if u == "all":
        app.unique = lambda step: True
    elif u is not None:
        us = set(u)
        app.unique = lambda step, us=us: step in us
    return app


def oracle_full_graph(dg) -> O.OGraph:
    """The whole device CSR copied to the host for the oracle."""
    h = dg.to_host()
    return O.OGraph(h.n_vertices, h.row_offsets, h.col_indices, h.weights,
                    h.per_vertex_weight_prefix, h.per_vertex_max_weight, None)


def oracle_subgraph(dg, vertices) -> O.OGraph:
    """An oracle graph with the device graph's rows of ``vertices`` only (every
    other row empty), gathered on the device so a 1B-edge graph never crosses
    to the host whole.  Sound for parity checks of runs whose transits are all
    in ``vertices``: where the device and the oracle agree the oracle reads
    exactly these rows, and where they first disagree the comparison fails
    (a missing row makes the oracle's sample differ, never agree)."""
    import torch
    a = dg.arrays()
    row = a["row_offsets"]
    V = dg.n_vertices
    v = torch.unique(torch.as_tensor(np.asarray(vertices, dtype=np.int64), device="cuda"))
    v = v[(v >= 0) & (v < V)]
    lo = row[v]
    deg = row[v + 1] - lo
    full = torch.zeros(V + 1, dtype=torch.int64, device="cuda")
    full[v + 1] = deg
    off = torch.cumsum(full, 0)
    seg = torch.repeat_interleave(torch.arange(len(v), device="cuda"), deg)
    start_new = off[v]
    pos = torch.arange(int(deg.sum().item()), device="cuda") - start_new[seg] + lo[seg]
    col = a["col"][pos].to(torch.int64)
    if dg.unit_weights:
        w = torch.ones(len(pos), dtype=torch.float64, device="cuda")
        pre = (pos - lo[seg] + 1).to(torch.float64)
    else:
        w, pre = a["weights"][pos], a["prefix"][pos]
    mx = torch.zeros(V, dtype=torch.float64, device="cuda")
    mx[v] = a["max_w"][v]
    return O.OGraph(V, off.cpu().numpy(), col.cpu().numpy(), w.cpu().numpy(), pre.cpu().numpy(),
                    mx.cpu().numpy(), None)


def expected_walk_rows(roots, r):
    """(offsets, ids) of walk final rows from an oracle run_chain result:
    row i = roots[i] then the chain's non-NULL vertices (chain.py:166-179)."""
    roots = np.asarray(roots, dtype=np.int64).reshape(len(r["chain_len"]), -1)
    clen, cv = np.asarray(r["chain_len"]), np.asarray(r["chain_vals"])
    starts = np.concatenate([[0], np.cumsum(clen)[:-1]]).astype(np.int64)
    ok = cv >= 0
    nn = np.add.reduceat(ok.astype(np.int64), starts) if len(cv) else np.zeros(len(clen), np.int64)
    nn = np.where(clen > 0, nn, 0)
    R = roots.shape[1]
    off = np.concatenate([[0], np.cumsum(R + nn)]).astype(np.int64)
    ids = np.empty(int(off[-1]), dtype=np.int64)
    is_root = np.zeros(len(ids), dtype=bool)
    for k in range(R):
        is_root[off[:-1] + k] = True
    ids[is_root] = roots.ravel()
    ids[~is_root] = cv[ok]
    return off, ids

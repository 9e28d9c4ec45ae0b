"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (needs /root/reference, read-only): the
reference package is copied to /tmp/trawl_ref, its Cython kernel is built
there (`python setup.py build_ext --inplace`, the reference's own recipe,
pkg/setup.py:5-27) and `trawl` is imported from it.  Nothing here is needed
on the GPU box — the fixtures it writes are committed.

    python tests/golden/make_golden.py

Fixtures:
  kat.json            RNG known answers, five-vertex batch vectors, class
                      thresholds, worker ranges
  batch_parity.npz    tests/test_kernels.py:58-74 pattern: 5000 random items
                      per app code on powerlaw(400, weighted, seed 8)
  graphs.npz          input graphs of the run fixtures (CSR arrays)
  runs.npz + runs.json  tp_run outputs (final rows, per-step rows, recorded
                      edges, stats) and sha256 of render_text per layout
  schedule.npz        build_transit_map / partition_work_classes exports
  csr_rmat.npz        reference from_edges on keyed RMAT edges (CSR pin)
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg"
REF_TMP = "/tmp/trawl_ref"


def import_reference():
    if not os.path.exists(os.path.join(REF_TMP, "src", "trawl")):
        shutil.copytree(REF_SRC, REF_TMP)
        subprocess.check_call(["chmod", "-R", "u+w", REF_TMP])
    so = [f for f in os.listdir(os.path.join(REF_TMP, "src", "trawl", "kernels"))
          if f.startswith("_ckernels") and f.endswith(".so")]
    if not so:
        subprocess.check_call([sys.executable, "setup.py", "build_ext", "--inplace"],
                              cwd=REF_TMP, stdout=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(REF_TMP, "src"))
    import trawl
    assert trawl.BACKEND_NAME == "compiled", trawl.BACKEND_NAME
    return trawl


def sha16(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()[:16]


def graph_arrays(prefix, g, store):
    store[f"{prefix}/row_offsets"] = g.row_offsets
    store[f"{prefix}/col_indices"] = g.col_indices
    store[f"{prefix}/weights"] = g.weights
    store[f"{prefix}/prefix"] = g.per_vertex_weight_prefix
    store[f"{prefix}/max_w"] = g.per_vertex_max_weight


def main():
    trawl = import_reference()
    from trawl import rng
    from trawl.apps import make_app
    from trawl.engine import EngineConfig, make_samples, tp_run, sp_run
    from trawl.engine.driver import StepPlan, worker_ranges
    from trawl.engine.transit_parallel import build_transit_map, partition_work_classes
    from trawl.graph import from_edges
    from trawl.kernels import _ckernels, K_DEEPWALK, K_PPR, K_NODE2VEC, K_KHOP, K_MULTIRW
    from trawl.output import render_text, LAYOUT_FINAL, LAYOUT_PER_STEP
    from trawl.synth import make_synthetic, powerlaw_graph, path_graph, star_graph, cycle_graph
    from trawl.core import Sample

    kat = {}
    # --- RNG known answers (SURVEY Appendix C + a sweep) -------------------
    keys = [(0, 0, 0, 0, 0, 0, 0), (7, 3, 2, 1, 4, 0, 9),
            (2**64 - 1, 10**6, 99, 24, 9, 1, 5), (123, 2**40, 10_000, 7, 3, 5, 2 * 999_999 + 1)]
    r = np.random.default_rng(0)
    for _ in range(40):
        keys.append((int(r.integers(0, 2**63)) * 2 + int(r.integers(0, 2)),
                     int(r.integers(0, 2**31)), int(r.integers(0, 10_000)),
                     int(r.integers(0, 1000)), int(r.integers(0, 1000)),
                     int(r.integers(0, 6)), int(r.integers(0, 1000))))
    kat["key_u64"] = [[list(k), str(rng.key_u64(*k)), rng.key_uniform(*k)] for k in keys]

    # --- five-vertex batch vectors (conftest.py:20-27) ----------------------
    g5 = from_edges([0, 0, 0, 0, 1, 1, 2], [1, 2, 3, 4, 0, 2, 3],
                    [1.5, 2.0, 0.5, 3.0, 1.0, 1.0, 1.0], n_vertices=5)
    kat["five_vertex"] = {"prefix": g5.per_vertex_weight_prefix.tolist(),
                          "max_w": g5.per_vertex_max_weight.tolist()}
    n = 8
    z = np.zeros(n, dtype=np.int64)
    sids = np.arange(n, dtype=np.int64)
    vec = {}
    for name, code, params, tprev in [
            ("deepwalk", K_DEEPWALK, [], -1), ("ppr", K_PPR, [0.3], -1),
            ("khop", K_KHOP, [], -1), ("multirw", K_MULTIRW, [], -1),
            ("node2vec", K_NODE2VEC, [2.0, 0.5, 0.0], 1),
            ("node2vec_direct", K_NODE2VEC, [2.0, 0.5, 1.0], 1)]:
        out = np.empty(n, dtype=np.int64)
        _ckernels.individual_batch(code, np.asarray(params, dtype=np.float64),
                                   g5.row_offsets, g5.col_indices, g5.weights,
                                   g5.per_vertex_weight_prefix, g5.per_vertex_max_weight,
                                   z.copy(), np.full(n, tprev, dtype=np.int64), sids, z, z,
                                   7, 1, out)
        vec[name] = out.tolist()
    kat["five_vertex"]["batch_seed7_step1"] = vec
    kat["worker_ranges"] = {f"{n_}_{w}": worker_ranges(n_, w)
                            for n_ in (0, 1, 7, 10, 100) for w in (1, 2, 3, 4, 8)}
    with open(os.path.join(HERE, "kat.json"), "w") as fh:
        json.dump(kat, fh, indent=1)

    # --- batch parity fixture (test_kernels.py:58-74 pattern) ---------------
    gp = powerlaw_graph(400, weighted=True, seed=8)
    store = {}
    graph_arrays("g", gp, store)
    params = {K_DEEPWALK: [], K_PPR: [0.05], K_NODE2VEC: [2.0, 0.5, 0.0],
              K_KHOP: [], K_MULTIRW: []}
    for code in sorted(params):
        rr = np.random.default_rng(code)
        N = 5000
        transits = rr.integers(0, gp.n_vertices, N).astype(np.int64)
        t_prev = np.full(N, -1, dtype=np.int64)
        if code == K_NODE2VEC:
            for i, v in enumerate(transits):
                nb = gp.neighbors(int(v))
                if len(nb) and rr.random() < 0.9:
                    t_prev[i] = int(nb.vertices[rr.integers(0, len(nb))])
        sids_ = rr.integers(0, 10_000, N).astype(np.int64)
        tix = rr.integers(0, 30, N).astype(np.int64)
        slots = rr.integers(0, 30, N).astype(np.int64)
        out = np.empty(N, dtype=np.int64)
        _ckernels.individual_batch(code, np.asarray(params[code], dtype=np.float64),
                                   gp.row_offsets, gp.col_indices, gp.weights,
                                   gp.per_vertex_weight_prefix, gp.per_vertex_max_weight,
                                   transits, t_prev, sids_, tix, slots, 123, 2, out)
        for k, v in dict(transits=transits, t_prev=t_prev, sample_ids=sids_,
                         transit_idxs=tix, slots=slots, out=out,
                         params=np.asarray(params[code], dtype=np.float64)).items():
            store[f"c{code}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "batch_parity.npz"), **store)

    # --- run fixtures ---------------------------------------------------------
    graphs = {}
    gstore = {}

    def G(spec, weighted, seed):
        key = f"{spec}|{int(weighted)}|{seed}"
        if key not in graphs:
            graphs[key] = make_synthetic(spec, weighted=weighted, seed=seed)
            graph_arrays(key, graphs[key], gstore)
        return key, graphs[key]

    runs_meta = []
    rstore = {}
    cases = [
        ("deepwalk", "cycle:200", False, 50, 7, {}),
        ("deepwalk", "powerlaw:2000", True, 500, 7, {}),
        ("ppr", "powerlaw:2000", True, 500, 7, {}),
        ("node2vec", "powerlaw:2000", True, 500, 7, {}),
        ("khop", "powerlaw:2000", False, 200, 3, {}),
        ("multirw", "powerlaw:2000", False, 50, 7, {}),
        ("layer", "powerlaw:2000", False, 8, 7, {}),
        ("fastgcn", "powerlaw:2000", False, 16, 7, {}),
        ("mvs", "powerlaw:2000", False, 16, 7, {}),
        ("clustergcn", "powerlaw:2000", False, 4, 7, {}),
    ]
    # cross-engine matrix (test_acceptance.py:46-69 shape, smaller graphs)
    per_app = {"deepwalk": 32, "ppr": 32, "node2vec": 32, "multirw": 12, "khop": 24,
               "layer": 8, "fastgcn": 12, "ladies": 12, "clustergcn": 4, "mvs": 16}
    for app_name, ns in per_app.items():
        for spec in ("path:300", "star:300", "powerlaw:1000"):
            for seed in (1, 2):
                cases.append((app_name, spec, True, ns, seed, {}))
    # parameter variants
    cases += [
        ("node2vec", "powerlaw:1000", True, 64, 5, {"factor_convention": "direct", "p": 0.5, "q": 2.0}),
        ("khop", "powerlaw:1000", True, 40, 5, {"fanouts": [5, 4, 3]}),
        ("ppr", "powerlaw:1000", True, 64, 9, {"termination_probability": 0.2}),
        ("fastgcn", "powerlaw:1000", False, 8, 4, {"distribution": "degree_sq"}),
        ("layer", "powerlaw:1000", False, 6, 4, {"max_size": 300, "step_size": 50}),
        ("multirw", "powerlaw:1000", True, 20, 4, {"roots_per_sample": 5, "walk_length": 30}),
        ("deepwalk", "path:300", True, 40, 3, {"walk_length": 400}),
        ("mvs", "powerlaw:1000", False, 8, 4, {"batch_size": 16, "step_size": 10}),
        ("clustergcn", "powerlaw:1000", False, 3, 4, {"clusters_per_sample": 5, "num_clusters": 20}),
    ]
    # unique()/dedup + SP-fallback routing (driver.py:165-172,
    # transit_parallel.py:200-231; tests/test_engines.py:194-215 pattern)
    cases += [
        ("khop", "cycle:200", True, 10, 14, {"fanouts": [12, 4], "unique": [0]}),
        ("khop", "powerlaw:1000", False, 30, 6, {"fanouts": [10, 5], "unique": "all"}),
        ("khop", "powerlaw:1000", False, 30, 6, {"fanouts": [25, 10], "unique": [1]}),
        ("khop", "star:300", True, 12, 2, {"fanouts": [40, 3], "unique": [0]}),
        ("layer", "powerlaw:1000", False, 6, 4, {"max_size": 300, "step_size": 50, "unique": "all"}),
        ("fastgcn", "powerlaw:1000", False, 6, 4, {"unique": [0, 2]}),
        ("mvs", "powerlaw:1000", False, 8, 4, {"batch_size": 16, "step_size": 40, "unique": "all"}),
    ]

    def apply_unique(app, kw):
        u = kw.get("unique")
        if u == "all":
            app.unique = lambda step: True
        elif u is not None:
            us = set(u)
            app.unique = lambda step, us=us: step in us
        return app

    for idx, (app_name, spec, weighted, ns, seed, kw) in enumerate(cases):
        gkey, g = G(spec, weighted, seed)
        mk = {k: v for k, v in kw.items() if k != "unique"}
        app = apply_unique(make_app(app_name, **mk), kw)
        samples = make_samples(app, g, ns, seed)
        out = tp_run(app, g, samples, EngineConfig(seed=seed))
        text_final = render_text(out, LAYOUT_FINAL)
        text_step = render_text(out, LAYOUT_PER_STEP)
        # SP must agree byte for byte (reference invariant)
        app2 = apply_unique(make_app(app_name, **mk), kw)
        out_sp = sp_run(app2, g, make_samples(app2, g, ns, seed), EngineConfig(seed=seed))
        assert render_text(out_sp, LAYOUT_FINAL) == text_final
        rows = out.final_rows()
        pre = f"r{idx}"
        rstore[f"{pre}/final_off"] = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
        rstore[f"{pre}/final_ids"] = (np.concatenate(rows) if rows else np.empty(0)).astype(np.int64)
        # per-step rows (non-NULL vertices per sample per step)
        steps_cnt, steps_ids = [], []
        for st in range(out.n_steps):
            rws = out.step_rows(st)
            steps_cnt.append([len(x) for x in rws])
            steps_ids.extend(np.concatenate(rws).tolist() if rws else [])
        rstore[f"{pre}/step_cnt"] = np.asarray(steps_cnt, dtype=np.int64).reshape(out.n_steps, ns)
        rstore[f"{pre}/step_ids"] = np.asarray(steps_ids, dtype=np.int64)
        rec_cnt, rec_t, rec_v = [], [], []
        if app.records_edges:
            for st in range(out.n_steps):
                row_c = []
                for s in out.samples:
                    if st < len(s.recorded_edges):
                        t_, v_ = s.recorded_edges[st]
                    else:
                        t_, v_ = np.empty(0, np.int64), np.empty(0, np.int64)
                    row_c.append(len(t_))
                    rec_t.extend(t_.tolist())
                    rec_v.extend(v_.tolist())
                rec_cnt.append(row_c)
        rstore[f"{pre}/rec_cnt"] = np.asarray(rec_cnt, dtype=np.int64).reshape(-1, ns)
        rstore[f"{pre}/rec_t"] = np.asarray(rec_t, dtype=np.int64)
        rstore[f"{pre}/rec_v"] = np.asarray(rec_v, dtype=np.int64)
        st = out.stats
        rstore[f"{pre}/groups"] = np.asarray(
            [[t.groups_small, t.groups_medium, t.groups_large] for t in st.timings],
            dtype=np.int64).reshape(-1, 3)
        runs_meta.append(dict(
            idx=idx, app=app_name, graph=gkey, weighted=weighted, n_samples=ns, seed=seed,
            params=kw, n_steps=out.n_steps, hash_final=sha16(text_final),
            hash_per_step=sha16(text_step), adjacency_fetches=st.adjacency_fetches,
            total_sampled=int(sum(s.total_sampled() for s in out.samples)),
            recorded=int(sum(sum(len(t_) for t_, _ in s.recorded_edges) for s in out.samples))))
    np.savez_compressed(os.path.join(HERE, "graphs.npz"), **gstore)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **rstore)
    with open(os.path.join(HERE, "runs.json"), "w") as fh:
        json.dump(runs_meta, fh, indent=1)

    # --- schedule fixtures (test_transit_schedule.py patterns) -------------
    sstore = {}
    sched_cases = [(50, (1, 8), 40, 1), (400, (5, 5), 60, 4), (2000, (50, 50), 500, 7),
                   (300, (1, 30), 3, 2), (64, (1, 3), 100000, 25)]
    for ci, (ns, (lo, hi), vmax, m) in enumerate(sched_cases):
        rr = np.random.default_rng(100 + ci)
        per = [rr.integers(0, vmax, size=int(rr.integers(lo, hi + 1))) for _ in range(ns)]
        app = make_app("khop", fanouts=[m])
        samples = [Sample(i, np.asarray(t, dtype=np.int64)) for i, t in enumerate(per)]
        plan = StepPlan(app, samples, 0, seed=0)
        groups = build_transit_map(plan)
        sched = partition_work_classes(groups, m)
        cls = {id(g): c for c, lst in enumerate((sched.small, sched.medium, sched.large)) for g in lst}
        sstore[f"s{ci}/pair_transit"] = plan.pair_transit
        sstore[f"s{ci}/m"] = np.asarray([m])
        sstore[f"s{ci}/order"] = np.concatenate([g.members for g in groups]).astype(np.int64)
        sstore[f"s{ci}/group_size"] = np.asarray([len(g.members) for g in groups], dtype=np.int64)
        sstore[f"s{ci}/group_transit"] = np.asarray([g.transit for g in groups], dtype=np.int64)
        sstore[f"s{ci}/group_class"] = np.asarray([cls[id(g)] for g in groups], dtype=np.int32)
        sstore[f"s{ci}/sched_index"] = np.asarray([sched.scheduling_index[g.transit] for g in groups],
                                                  dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "schedule.npz"), **sstore)

    # --- CSR pin: reference from_edges on keyed RMAT edges -----------------
    sys.path.insert(0, REPO)
    from oracle import oracle as O
    cstore = {}
    for scale, ef, und, wt in [(9, 8, False, True), (8, 4, True, False), (10, 16, False, True)]:
        src, dst, w = O.rmat_edges(scale, (1 << scale) * ef, seed=scale, undirected=und, weighted=wt)
        gref = from_edges(src, dst, w if wt else None, n_vertices=1 << scale)
        k = f"s{scale}_{ef}_{int(und)}_{int(wt)}"
        cstore[f"{k}/src"] = src
        cstore[f"{k}/dst"] = dst
        cstore[f"{k}/w"] = w
        graph_arrays(k, gref, cstore)
    np.savez_compressed(os.path.join(HERE, "csr_rmat.npz"), **cstore)
    print("golden fixtures written:", len(runs_meta), "runs")


if __name__ == "__main__":
    main()

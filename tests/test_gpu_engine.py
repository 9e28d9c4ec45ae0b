"""End-to-end parity of the device engine (tp_run / sp_run through the
C-ABI) against the reference's golden hashes and the C oracle."""

import os
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import build_app, golden, golden_graph, oracle_run, recorded_equal, sha16, texts

pytestmark = pytest.mark.gpu

WALKS = ("deepwalk", "ppr", "node2vec", "multirw")


def _cases(apps):
    return [m for m in golden("runs.json") if m["app"] in apps]


def _device_run(meta, paradigm):
    from paper_2009_06693_b200 import EngineConfig, make_app, make_samples, sp_run, tp_run
    from paper_2009_06693_b200.graph import DeviceGraph
    g = golden_graph(meta["graph"])
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    app = build_app(meta)
    samples = make_samples(app, g, meta["n_samples"], meta["seed"])
    run = tp_run if paradigm == "tp" else sp_run
    return run(app, dg, samples, EngineConfig(seed=meta["seed"]))


@pytest.mark.parametrize("paradigm", ["tp", "tp-classes", "sp"])
@pytest.mark.parametrize("meta", _cases(WALKS), ids=lambda m: f"{m['idx']}-{m['app']}-{m['graph']}")
def test_walk_runs_match_reference(meta, paradigm, monkeypatch):
    # "tp": golden runs are small, so every step runs in the TP tail (walker-major
    # windows + class statistics from the logged transits); "tp-classes": every
    # step through the TP class kernels (ND_TP_TAIL=0)
    if paradigm == "tp-classes":
        monkeypatch.setenv("ND_TP_TAIL", "0")
        paradigm = "tp"
    out = _device_run(meta, paradigm)
    tf, ts = texts(out)
    assert out.n_steps == meta["n_steps"]
    assert sha16(tf) == meta["hash_final"]
    assert sha16(ts) == meta["hash_per_step"]
    assert out.total_sampled() == meta["total_sampled"]
    if paradigm == "tp":
        rs = golden("runs.npz")
        groups = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in out.stats.timings])
        assert np.array_equal(groups.reshape(-1, 3), rs[f"r{meta['idx']}/groups"])
        assert out.stats.adjacency_fetches == meta["adjacency_fetches"]


def test_device_graph_roundtrip_and_unit_detection():
    from paper_2009_06693_b200.graph import DeviceGraph
    g = golden_graph("powerlaw:2000|0|7")
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    assert dg.unit_weights
    h = dg.to_host()
    assert np.array_equal(h.row_offsets, g.row_offsets)
    assert np.array_equal(h.col_indices, g.col_indices)
    assert np.array_equal(h.per_vertex_max_weight, g.per_vertex_max_weight)
    gw = golden_graph("powerlaw:2000|1|7")
    dw = DeviceGraph.from_arrays(gw.row_offsets, gw.col_indices, gw.weights)
    assert not dw.unit_weights
    hw = dw.to_host()
    assert np.array_equal(hw.per_vertex_weight_prefix, gw.per_vertex_weight_prefix)
    assert np.array_equal(hw.per_vertex_max_weight, gw.per_vertex_max_weight)


@pytest.mark.parametrize("key", ["s9_8_0_1", "s8_4_1_0", "s10_16_0_1"])
def test_device_rmat_matches_reference_from_edges(key):
    """Device RMAT generation + CSR build == the reference from_edges on the
    same keyed edges (golden csr_rmat.npz)."""
    from paper_2009_06693_b200.graph import DeviceGraph
    d = golden("csr_rmat.npz")
    scale, ef, und, wt = (int(x) for x in key[1:].split("_"))
    dg = DeviceGraph.rmat(scale, ef, seed=scale, undirected=bool(und), weighted=bool(wt))
    h = dg.to_host()
    assert np.array_equal(h.row_offsets, d[f"{key}/row_offsets"])
    assert np.array_equal(h.col_indices, d[f"{key}/col_indices"])
    if wt:
        assert np.array_equal(h.weights, d[f"{key}/weights"])
        assert np.array_equal(h.per_vertex_weight_prefix, d[f"{key}/prefix"])
    assert np.array_equal(h.per_vertex_max_weight, d[f"{key}/max_w"])
    # device from_edges on the same edge list
    de = DeviceGraph.from_edges(d[f"{key}/src"], d[f"{key}/dst"], d[f"{key}/w"] if wt else None,
                                1 << scale)
    he = de.to_host()
    assert np.array_equal(he.row_offsets, d[f"{key}/row_offsets"])
    assert np.array_equal(he.col_indices, d[f"{key}/col_indices"])


@pytest.mark.parametrize("app,params,weighted", [
    ("deepwalk", {}, True), ("deepwalk", {}, False), ("ppr", {}, True),
    ("node2vec", {}, True), ("node2vec", {}, False), ("multirw", {"roots_per_sample": 8}, False),
    # factor orders that move the membership band (n2v_accept): f_adj > f_far,
    # the direct convention, and p = q = 1 (empty band: never probed)
    ("node2vec", {"p": 0.5, "q": 2.0, "walk_length": 40}, True),
    ("node2vec", {"p": 2.0, "q": 0.5, "factor_convention": "direct", "walk_length": 40}, True),
    ("node2vec", {"p": 1.0, "q": 1.0, "walk_length": 40}, True)])
def test_walks_on_rmat_vs_oracle(app, params, weighted):
    """Scale-14 RMAT (skewed degrees, zero-degree vertices, hubs that land in
    the medium/large TP classes): device == multi-threaded oracle, bit for bit,
    plus the TP class statistics of a single-thread oracle."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    scale, n = 14, 20_000
    dg = DeviceGraph.rmat(scale, 16, seed=5, weighted=weighted)
    hg = dg.to_host()
    og = O.OGraph(hg.n_vertices, hg.row_offsets, hg.col_indices, hg.weights,
                  hg.per_vertex_weight_prefix, hg.per_vertex_max_weight, np.arange(hg.n_vertices))
    a = make_app(app, **params)
    meta = {"app": app, "params": params, "n_samples": n, "seed": 9}
    ref = oracle_run(meta, og, paradigm="tp", n_threads=1)
    # TP with every step in the class kernels, with the hand-off to the
    # walker-major tail mid-run, and with the default threshold (all tail)
    for par, tail in (("tp", "0"), ("tp", "5000"), ("tp", None), ("sp", None)):
        if tail is None:
            os.environ.pop("ND_TP_TAIL", None)
        else:
            os.environ["ND_TP_TAIL"] = tail
        try:
            dr = run_device(a, dg, n_samples=n, seed=9, paradigm=par)
        finally:
            os.environ.pop("ND_TP_TAIL", None)
        out = dr.to_output()
        off, ids = out.final_csr()
        roff, rids = ref.final_csr()
        assert np.array_equal(off, roff) and np.array_equal(ids, rids), (par, tail)
        assert out.n_steps == ref.n_steps
        if par == "tp":
            st = dr.stats()
            got = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in st.timings])
            assert np.array_equal(got.reshape(-1, 3), ref.stats[:, :3])
            assert st.adjacency_fetches == int(ref.stats[:, 3].sum())
        dr.close()


@pytest.mark.parametrize("paradigm", ["tp", "sp"])
@pytest.mark.parametrize("meta", _cases(("khop",)), ids=lambda m: f"{m['idx']}-{m['app']}-{m['graph']}")
def test_khop_runs_match_reference(meta, paradigm):
    out = _device_run(meta, paradigm)
    tf, ts = texts(out)
    assert out.n_steps == meta["n_steps"]
    assert sha16(tf) == meta["hash_final"]
    assert sha16(ts) == meta["hash_per_step"]
    if paradigm == "tp":
        rs = golden("runs.npz")
        groups = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in out.stats.timings])
        assert np.array_equal(groups.reshape(-1, 3), rs[f"r{meta['idx']}/groups"])
        assert out.stats.adjacency_fetches == meta["adjacency_fetches"]


def test_khop_on_rmat_vs_oracle():
    """Reddit-shaped (symmetric RMAT, unit weights) 2-hop 25/10 on 3000 roots:
    device == oracle for every step slot, final rows and TP class counts."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(13, 16, seed=3, undirected=True, weighted=False)
    hg = dg.to_host()
    og = O.OGraph(hg.n_vertices, hg.row_offsets, hg.col_indices, hg.weights,
                  hg.per_vertex_weight_prefix, hg.per_vertex_max_weight, np.arange(hg.n_vertices))
    meta = {"app": "khop", "params": {}, "n_samples": 3000, "seed": 4}
    ref = oracle_run(meta, og, paradigm="tp")
    for par in ("tp", "sp"):
        dr = run_device(make_app("khop"), dg, n_samples=3000, seed=4, paradigm=par)
        out = dr.to_output()
        assert np.array_equal(out.step_counts, ref.step_counts)
        assert np.array_equal(out.step_vals, ref.step_vals)
        off, ids = out.final_csr()
        roff, rids = ref.final_csr()
        assert np.array_equal(off, roff) and np.array_equal(ids, rids)
        if par == "tp":
            st = dr.stats()
            got = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in st.timings])
            assert np.array_equal(got.reshape(-1, 3), ref.stats[:, :3])
        dr.close()


@pytest.mark.parametrize("ci", range(5))
def test_schedule_export_matches_reference(ci):
    from paper_2009_06693_b200.schedule import transit_schedule
    d = golden("schedule.npz")
    r = transit_schedule(d[f"s{ci}/pair_transit"], int(d[f"s{ci}/m"][0]))
    assert np.array_equal(r["order"], d[f"s{ci}/order"])
    assert np.array_equal(np.diff(r["group_start"]), d[f"s{ci}/group_size"])
    assert np.array_equal(r["group_transit"], d[f"s{ci}/group_transit"])
    assert np.array_equal(r["group_class"], d[f"s{ci}/group_class"])
    assert np.array_equal(r["sched_index"], d[f"s{ci}/sched_index"])


def test_reference_app_objects_accepted():
    """A reference-shaped app (duck-typed SamplingApp with kernel_code and
    params, closure-based init_roots) runs unchanged."""
    from paper_2009_06693_b200 import EngineConfig, tp_run
    from paper_2009_06693_b200.core import INDIVIDUAL, SamplingApp
    from paper_2009_06693_b200.engine import make_samples
    from paper_2009_06693_b200.graph import DeviceGraph
    meta = [m for m in golden("runs.json") if m["app"] == "deepwalk" and m["graph"].startswith("powerlaw:2000")][0]
    g = golden_graph(meta["graph"])

    def init(graph, sid, seed):  # the reference's closure shape (apps.py:83-103)
        from paper_2009_06693_b200.apps import UniformRoots
        return UniformRoots(1)(graph, sid, seed)

    app = SamplingApp(name="deepwalk", sampling_type=INDIVIDUAL, steps=100,
                      sample_size=lambda s: 1, next_fn=lambda *a: -1, init_roots=init,
                      chain_walk=True, kernel_code=0, params={"walk_length": 100})
    samples = [make_samples(app, g, meta["n_samples"], meta["seed"])[i] for i in range(meta["n_samples"])]
    out = tp_run(app, DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights), samples,
                 EngineConfig(seed=meta["seed"]))
    assert sha16(texts(out)[0]) == meta["hash_final"]


COLLECTIVE = ("layer", "fastgcn", "ladies", "mvs", "clustergcn")


@pytest.mark.parametrize("meta", _cases(COLLECTIVE), ids=lambda m: f"{m['idx']}-{m['app']}-{m['graph']}")
def test_collective_runs_match_reference(meta):
    out = _device_run(meta, "tp")
    tf, ts = texts(out)
    assert out.n_steps == meta["n_steps"]
    assert sha16(tf) == meta["hash_final"]
    assert sha16(ts) == meta["hash_per_step"]
    rs = golden("runs.npz")
    assert recorded_equal(out, rs, f"r{meta['idx']}")
    assert out.total_recorded() == meta["recorded"]
    groups = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in out.stats.timings])
    assert np.array_equal(groups.reshape(-1, 3), rs[f"r{meta['idx']}/groups"])
    assert out.stats.adjacency_fetches == meta["adjacency_fetches"]


@pytest.mark.parametrize("app,params", [("fastgcn", {}), ("ladies", {"distribution": "degree_sq"}),
                                        ("mvs", {}), ("layer", {"max_size": 500, "step_size": 100}),
                                        ("clustergcn", {"clusters_per_sample": 3, "num_clusters": 10})])
def test_collective_on_rmat_vs_oracle(app, params):
    """Orkut-shaped (symmetric RMAT, unit weights) collective sampling at scale 12
    vs the oracle: slots, recorded edges, final rows."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(12, 16, seed=8, undirected=True, weighted=False)
    hg = dg.to_host()
    og = O.OGraph(hg.n_vertices, hg.row_offsets, hg.col_indices, hg.weights,
                  hg.per_vertex_weight_prefix, hg.per_vertex_max_weight, np.arange(hg.n_vertices))
    n = 6 if app == "clustergcn" else 96
    meta = {"app": app, "params": params, "n_samples": n, "seed": 12}
    ref = oracle_run(meta, og)
    dr = run_device(make_app(app, **params), dg, n_samples=n, seed=12)
    out = dr.to_output()
    assert out.n_steps == ref.n_steps
    assert np.array_equal(out.step_counts, ref.step_counts)
    assert np.array_equal(out.step_vals, ref.step_vals)
    if app != "layer":  # layer records no edges (apps.py:247-283)
        assert np.array_equal(np.asarray(out.rec_counts), np.asarray(ref.rec_counts))
        assert np.array_equal(out.rec_t, ref.rec_t) and np.array_equal(out.rec_v, ref.rec_v)
    else:
        assert out.rec_t is None and len(ref.rec_t) == 0
    off, ids = out.final_csr()
    roff, rids = ref.final_csr()
    assert np.array_equal(off, roff) and np.array_equal(ids, rids)
    dr.close()


def _hub_graph(V=3000, hub_deg=5000):
    """Vertex 0 a hub of hub_deg out-edges; every other vertex a few edges
    back to the hub and to random vertices; weights spanning six decades with
    10% zeros; parallel edges kept."""
    rng = np.random.default_rng(21)
    src = [np.zeros(hub_deg, dtype=np.int64)]
    dst = [rng.integers(1, V, hub_deg)]
    for v in range(1, V):
        k = int(rng.integers(1, 60))
        src.append(np.full(k, v))
        d = rng.integers(0, V, k)
        d[0] = 0
        dst.append(d)
    src, dst = np.concatenate(src), np.concatenate(dst)
    w = 10.0 ** rng.uniform(-3, 3, len(src))
    w[rng.random(len(src)) < 0.1] = 0.0
    return O.from_edges(src, dst, w, V)


@pytest.mark.parametrize("app,params", [("clustergcn", {"clusters_per_sample": 3, "num_clusters": 7}),
                                        ("mvs", {}), ("fastgcn", {}), ("layer", {})])
def test_collective_on_hub_graph_vs_oracle(app, params):
    """Collective apps where one transit's row (5,000 edges) spans several
    of ClusterGCN's 1,024-edge scan units and many transits have short rows:
    slots, recorded edges (order included) and final rows == oracle, both
    paradigms."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    og = _hub_graph()
    dg = DeviceGraph.from_arrays(og.row_offsets, og.col_indices, og.weights)
    n = 5 if app == "clustergcn" else 64
    meta = {"app": app, "params": params, "n_samples": n, "seed": 4}
    ref = oracle_run(meta, og)
    for par in ("sp", "tp"):
        dr = run_device(make_app(app, **params), dg, n_samples=n, seed=4, paradigm=par)
        out = dr.to_output()
        assert np.array_equal(out.step_vals, ref.step_vals), par
        if app != "layer":
            assert np.array_equal(np.asarray(out.rec_counts), np.asarray(ref.rec_counts)), par
            assert np.array_equal(out.rec_t, ref.rec_t) and np.array_equal(out.rec_v, ref.rec_v), par
        off, ids = out.final_csr()
        roff, rids = ref.final_csr()
        assert np.array_equal(off, roff) and np.array_equal(ids, rids), par
        dr.close()


@pytest.mark.parametrize("app", ["deepwalk", "ppr", "node2vec"])
def test_index_paths_on_adversarial_hub_graph(app):
    """Guide-table picks and hash-set membership on rows far above the index
    thresholds, with zero weights (flat prefix runs), weights spanning six
    decades, parallel edges and a dense hub neighbourhood: device == oracle."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    og = _hub_graph()
    dg = DeviceGraph.from_arrays(og.row_offsets, og.col_indices, og.weights)
    n = 4000
    meta = {"app": app, "params": {}, "n_samples": n, "seed": 33}
    ref = oracle_run(meta, og)
    for par in ("sp", "tp"):
        dr = run_device(make_app(app), dg, n_samples=n, seed=33, paradigm=par)
        off, ids = dr.host(0), dr.host(1)
        roff, rids = ref.final_csr()
        assert np.array_equal(off, roff) and np.array_equal(ids, rids), par
        dr.close()


def test_unique_fallback_routing_object_mode():
    """tests/test_engines.py:194-215 of the reference: an object-mode k-hop
    (kernel_code None) with a unique first step on a degree-1 cycle: every
    sample dedups to one vertex, is flagged for the SP fallback, and TP/SP
    outputs agree."""
    from paper_2009_06693_b200 import EngineConfig, make_app, make_samples, sp_run, tp_run
    from paper_2009_06693_b200.synth import cycle_graph
    g = cycle_graph(40, weighted=True, seed=2)

    def build():
        app = make_app("khop", fanouts=[12, 4])
        app.unique = lambda step: step == 0
        app.kernel_code = None
        return app

    texts_ = {}
    for run, label in [(sp_run, "sp"), (tp_run, "tp")]:
        app = build()
        out = run(app, g, make_samples(app, g, 10, seed=14), EngineConfig(seed=14))
        assert all(len(s.vertices_at(0)) == 1 for s in out.samples)
        assert all(len(s.vertices_at(1)) == 4 for s in out.samples)
        texts_[label] = texts(out)[0]
        if label == "tp":
            # all 10 samples flagged: step 1 runs sample-parallel, no TP groups
            t1 = out.stats.timings[1]
            assert (t1.groups_small, t1.groups_medium, t1.groups_large) == (0, 0, 0)
    assert texts_["sp"] == texts_["tp"]


def test_custom_init_roots_star_single_giant_group():
    """tests/test_engines.py:218-228: custom init_roots (every sample rooted
    at the hub) -> one TP group at step 0, classed medium (work 60)."""
    from paper_2009_06693_b200 import EngineConfig, make_app, make_samples, tp_run
    from paper_2009_06693_b200.synth import star_graph
    g = star_graph(200)
    app = make_app("khop", fanouts=[2, 2])
    app.init_roots = lambda graph, sid, seed: np.asarray([0], dtype=np.int64)
    out = tp_run(app, g, make_samples(app, g, 30, seed=1), EngineConfig(seed=1))
    t0 = out.stats.timings[0]
    assert (t0.groups_small + t0.groups_medium + t0.groups_large) == 1
    assert t0.groups_medium == 1
    assert all(r[0] == 0 for r in out.final_rows())


@pytest.mark.parametrize("case", golden("cli.json"), ids=lambda c: "-".join(c["args"][1:2] + c["args"][3:4]))
def test_cli_output_matches_reference_cli(case, tmp_path):
    """The device CLI writes the reference CLI's bytes (output text, .remap
    sidecar) and the same deterministic report keys (cli.py:88-137)."""
    import hashlib
    from paper_2009_06693_b200.cli import main
    o, r = tmp_path / "out.txt", tmp_path / "rep.txt"
    assert main([*case["args"], "--output", str(o), "--report", str(r)]) == 0
    sha = lambda p: hashlib.sha256(open(p, "rb").read()).hexdigest()[:16]
    assert sha(o) == case["output"]
    assert sha(str(o) + ".remap") == case["remap"]
    rep = dict(line.split("=", 1) for line in open(r).read().splitlines())
    for k, v in case["report"].items():
        assert rep[k] == v, k


def test_narrowed_ids_match_int64_rows():
    """nd_result_narrow_ids: the int32 final ids (the e2e D2H payload) equal the
    int64 final ids element for element, and host copies of both agree."""
    import torch
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(12, 16, seed=3, weighted=True)
    for app in ("node2vec", "ppr", "khop"):
        dr = run_device(make_app(app), dg, n_samples=3001, seed=4, paradigm="sp")
        v32 = dr.narrow_ids()
        assert v32.dtype == torch.int32
        assert dr.narrow_ids().data_ptr() == v32.data_ptr()  # idempotent
        ids64 = dr.host(_lib.F_FINAL_IDS)
        ids32 = dr.host(_lib.F_FINAL_IDS32)
        assert ids32.dtype == np.int32 and np.array_equal(ids32.astype(np.int64), ids64)
        assert torch.equal(v32.to(torch.int64), dr.view(_lib.F_FINAL_IDS))
        dr.close()


def test_concurrent_jobs_and_host_pipeline_match_plain_runs():
    """run_device_concurrent (one stream + host thread per job) and the chunked
    HostPipeline return exactly the rows of plain sequential runs."""
    import torch
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device, run_device_concurrent
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.streaming import HostPipeline
    dg = DeviceGraph.rmat(13, 16, seed=11, weighted=True)
    apps = [make_app("node2vec"), make_app("ppr"), make_app("deepwalk")]
    n, seed = 5000, 3
    ref = []
    for a in apps:
        dr = run_device(a, dg, n_samples=n, sample_lo=17, seed=seed, paradigm="sp")
        ref.append((dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)))
        dr.close()
    runs = run_device_concurrent([dict(app=a, n_samples=n, sample_lo=17, seed=seed) for a in apps], dg)
    torch.cuda.synchronize()
    for dr, (off, ids) in zip(runs, ref):
        assert np.array_equal(dr.host(_lib.F_FINAL_OFF), off)
        assert np.array_equal(dr.host(_lib.F_FINAL_IDS), ids)
        dr.close()
    for chunks in (1, 3):
        pipe = HostPipeline(chunks=chunks)
        res = pipe.run_jobs(dg, [(a, n, seed, 17, None) for a in apps])
        for parts, (off, ids) in zip(res, ref):
            got_ids = np.concatenate([c.ids.numpy().astype(np.int64) for c in parts])
            got_len = np.concatenate([np.diff(c.offsets.numpy()) for c in parts])
            assert np.array_equal(got_ids, ids) and np.array_equal(got_len, np.diff(off))
            assert sum(c.n for c in parts) == n and parts[0].sample_lo == 17
    # explicit host roots shared by the walk jobs (uploaded once, before sampling),
    # weighted chunk plans, and the old per-chunk upload: rows equal plain runs
    rng = np.random.default_rng(4)
    roots = torch.from_numpy(rng.integers(0, dg.n_vertices, n)).pin_memory()
    ref2 = []
    for a in apps:
        droots = roots.to("cuda")
        from paper_2009_06693_b200.streaming import _run_walk_with_roots
        from paper_2009_06693_b200.engine import describe
        dr = _run_walk_with_roots(describe(a), dg, droots, 1, 17, n, seed, "sp", 10_000)
        ref2.append((dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)))
        dr.close()
    for mode, spec in ((None, 3), (None, (1, 5, 5, 2)), ("chunk", 2)):
        if mode:
            os.environ["ND_PIPE_ROOTS"] = mode
        try:
            pipe = HostPipeline(chunks=3)
            res = pipe.run_jobs(dg, [(a, n, seed, 17, roots, spec) for a in apps])
        finally:
            os.environ.pop("ND_PIPE_ROOTS", None)
        assert pipe.last_h2d_bytes == n * 8 * (len(apps) if mode else 1)
        if mode is None and spec == 3:  # back-to-back runs: both results valid after wait()
            pipe2 = HostPipeline(chunks=3)
            r1 = pipe2.run_jobs(dg, [(a, n, seed, 17, roots, 3) for a in apps], wait=False)
            r2 = pipe2.run_jobs(dg, [(a, n, seed, 17, roots, 2) for a in apps], wait=False)
            pipe2.wait()
            for rr in (r1, r2):
                for parts, (off, ids) in zip(rr, ref2):
                    got = np.concatenate([c.ids.numpy().astype(np.int64) for c in parts])
                    assert np.array_equal(got, ids)
        for parts, (off, ids) in zip(res, ref2):
            got_ids = np.concatenate([c.ids.numpy().astype(np.int64) for c in parts])
            got_len = np.concatenate([np.diff(c.offsets.numpy()) for c in parts])
            assert np.array_equal(got_ids, ids) and np.array_equal(got_len, np.diff(off)), (mode, spec)


def test_final_samples_dense_matches_rows():
    """DeviceRun.final_samples (the frontend's getFinalSamples): dense int32
    rows padded with -1, equal to the final rows; exported through DLPack."""
    import torch
    from torch.utils.dlpack import from_dlpack, to_dlpack
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(12, 16, seed=2, weighted=True)
    for app in ("ppr", "khop", "fastgcn"):
        dr = run_device(make_app(app), dg, n_samples=777, seed=5, paradigm="sp" if app != "fastgcn" else "tp")
        off, ids = dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)
        dense = dr.final_samples()
        width = int(np.diff(off).max())
        assert dense.shape == (777, width) and dense.dtype == torch.int32
        d = from_dlpack(to_dlpack(dense)).cpu().numpy()
        for i in range(777):
            row = ids[off[i]:off[i + 1]]
            assert np.array_equal(d[i, :len(row)], row) and (d[i, len(row):] == -1).all()
        dr.close()


@pytest.mark.parametrize("par,R,fan", [("sp", 3, "6,4"), ("tp", 3, "6,4"), ("sp", 2, "4,3,2"),
                                       ("tp", 1, "3,3,3,2")])
def test_fixed_layout_matches_step_loop(par, R, fan, tmp_path):
    """The fixed-layout k-hop (per-sample blocks, no host sync between steps)
    against the step-loop engine (ND_IND_FIXED=0) on a directed RMAT graph with
    dead ends: several roots per sample and 3-4 hops; final rows, step rows,
    TP class counts and adjacency fetches equal."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    helper = os.path.join(repo, "tests", "_khop_engine_dump.py")
    res = {}
    for fixed in ("1", "0"):
        path = str(tmp_path / f"r{fixed}.npz")
        env = dict(os.environ, ND_IND_FIXED=fixed)
        subprocess.check_call([sys.executable, helper, repo, path, par, str(R), fan], env=env)
        res[fixed] = np.load(path)
    a, b = res["1"], res["0"]
    for k in ("off", "ids", "sc", "sv", "n_steps", "fetch"):
        assert np.array_equal(a[k], b[k]), k
    if par == "tp":
        assert np.array_equal(a["cls"], b["cls"])


def _final_equal(dr, ref, tag):
    out = dr.to_output()
    off, ids = out.final_csr()
    roff, rids = ref.final_csr()
    assert np.array_equal(off, roff) and np.array_equal(ids, rids), tag
    assert out.n_steps == ref.n_steps, tag
    return out


@pytest.mark.parametrize("app,params", [("ppr", {}), ("node2vec", {"walk_length": 30}),
                                        ("deepwalk", {}), ("multirw", {"roots_per_sample": 4})])
def test_step_cap_and_tp_tail_vs_oracle(app, params):
    """Walks cut by a small step cap (INF-length PPR reaches it inside the
    walker-major windows), for SP, TP in the class kernels, TP handing off to
    the tail mid-run and TP all tail: rows, n_steps and TP class counts equal
    the oracle's."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(12, 16, seed=3, weighted=app != "multirw")
    hg = dg.to_host()
    og = O.OGraph(hg.n_vertices, hg.row_offsets, hg.col_indices, hg.weights,
                  hg.per_vertex_weight_prefix, hg.per_vertex_max_weight, np.arange(hg.n_vertices))
    n, cap = 3000, 9
    meta = {"app": app, "params": params, "n_samples": n, "seed": 9}
    ref = oracle_run(meta, og, paradigm="tp", step_cap=cap)
    a = make_app(app, **params)
    for par, tail in (("sp", None), ("tp", "0"), ("tp", "300"), ("tp", None)):
        if tail is not None:
            os.environ["ND_TP_TAIL"] = tail
        try:
            dr = run_device(a, dg, n_samples=n, seed=9, paradigm=par, step_cap=cap)
        finally:
            os.environ.pop("ND_TP_TAIL", None)
        _final_equal(dr, ref, (app, par, tail))
        if par == "tp":
            st = dr.stats()
            got = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in st.timings])
            assert np.array_equal(got.reshape(-1, 3), ref.stats[:, :3]), (app, tail)
        dr.close()


def test_edgeless_graph_and_empty_jobs():
    """A graph with vertices and no edges (every walk and hop ends at its
    root; collective steps find nothing), and zero-sample jobs for every app
    and paradigm."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    V = 64
    dg0 = DeviceGraph.from_arrays(np.zeros(V + 1, dtype=np.int64), np.zeros(0, dtype=np.int64))
    hg = dg0.to_host()
    og = O.OGraph(hg.n_vertices, hg.row_offsets, hg.col_indices, hg.weights,
                  hg.per_vertex_weight_prefix, hg.per_vertex_max_weight, np.arange(V))
    dg = DeviceGraph.rmat(10, 8, seed=1, weighted=True)
    cases = [("deepwalk", {}), ("ppr", {}), ("node2vec", {}), ("multirw", {"roots_per_sample": 4}),
             ("khop", {}), ("layer", {"max_size": 40, "step_size": 8}), ("fastgcn", {}), ("mvs", {})]
    for app, params in cases:
        a = make_app(app, **params)
        meta = {"app": app, "params": params, "n_samples": 40, "seed": 5}
        ref = oracle_run(meta, og, paradigm="tp")
        for par in ("sp", "tp"):
            dr = run_device(a, dg0, n_samples=40, seed=5, paradigm=par)
            out = dr.to_output()
            off, ids = out.final_csr()
            roff, rids = ref.final_csr()
            assert np.array_equal(off, roff) and np.array_equal(ids, rids), (app, par)
            assert dr.total_sampled == ref.total_sampled(), (app, par, dr.total_sampled,
                                                             ref.total_sampled())
            dr.close()
            dr = run_device(a, dg, n_samples=0, seed=5, paradigm=par)
            assert dr.total_sampled == 0, (app, par)
            assert list(dr.to_output().final_csr()[0]) == [0], (app, par)
            dr.close()


@pytest.mark.parametrize("paradigm", ["tp", "sp"])
def test_unbounded_app_step_cap_warns(paradigm):
    """An INF-step app that reaches the step cap warns like run_chain/run_loop
    (chain.py:93-98, driver.py:215-220; reference test_engines.py:173-178)."""
    from paper_2009_06693_b200 import EngineConfig, make_app, make_samples, sp_run, tp_run
    from paper_2009_06693_b200.synth import cycle_graph
    g = cycle_graph(1000, weighted=True, seed=2)
    app = make_app("ppr", termination_probability=0.0001)  # walks outlive the cap
    run = tp_run if paradigm == "tp" else sp_run
    with pytest.warns(RuntimeWarning, match="step cap"):
        out = run(app, g, make_samples(app, g, 4, seed=1), EngineConfig(seed=1, step_cap=50))
    assert out.n_steps == 50


@pytest.mark.parametrize("paradigm", ["sp", "tp"])
def test_gpu_share_keeps_rows(paradigm):
    """Runs started under engine.gpu_share(k) (nd_set_concurrency: persistent
    kernels take 1/k of every SM's CTA slots, walk kernels built for 4 CTAs
    per SM) return the rows of whole-GPU runs."""
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import gpu_share, run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(13, 16, seed=11, weighted=True)
    for name in ("node2vec", "ppr", "deepwalk"):
        app = make_app(name)
        dr = run_device(app, dg, n_samples=6000, seed=5, paradigm=paradigm)
        ref = (dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS))
        dr.close()
        for k in (2, 3, 8):
            with gpu_share(k):
                dr = run_device(app, dg, n_samples=6000, seed=5, paradigm=paradigm)
            assert np.array_equal(dr.host(_lib.F_FINAL_OFF), ref[0])
            assert np.array_equal(dr.host(_lib.F_FINAL_IDS), ref[1])
            dr.close()


def test_big_graph_walk_grid_keeps_rows(monkeypatch):
    """Graphs above ND_WALK_BIG_GB run the walk kernel at 2 CTAs per SM
    (forced here on a small graph): rows equal the default grid's."""
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(13, 16, seed=11, weighted=True)
    for name in ("node2vec", "ppr", "deepwalk"):
        app = make_app(name)
        dr = run_device(app, dg, n_samples=6000, seed=5, paradigm="sp")
        ref = (dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS))
        dr.close()
        monkeypatch.setenv("ND_WALK_BIG_GB", "0.000001")
        dr = run_device(app, dg, n_samples=6000, seed=5, paradigm="sp")
        monkeypatch.delenv("ND_WALK_BIG_GB")
        assert np.array_equal(dr.host(_lib.F_FINAL_OFF), ref[0])
        assert np.array_equal(dr.host(_lib.F_FINAL_IDS), ref[1])
        dr.close()


@pytest.mark.parametrize("env", [{}, {"ND_TP_TAIL": "0"}, {"ND_TP_TAIL": "0", "ND_TW_STAGE": "0"},
                                 {"ND_TP_TAIL": "0", "ND_TW_STAGE": "0", "ND_TW_MULTI": "1"}],
                         ids=["tail", "hub", "multi", "one-step"])
@pytest.mark.parametrize("paradigm", ["sp", "tp"])
def test_node2vec_stall_raises(paradigm, env, monkeypatch):
    """node2vec whose acceptance is ~0 (p = q = 1e300) exhausts its tries on
    the second step and the run raises SamplerStallError (chain.py stall
    contract), in every walk engine: walker-major, TP tail, TP hub steps,
    K-step TP launches and one-step TP launches."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.errors import SamplerStallError
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.synth import cycle_graph
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = cycle_graph(64, weighted=True, seed=1)
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    app = make_app("node2vec", p=1e300, q=1e300)
    with pytest.raises(SamplerStallError):
        dr = run_device(app, dg, n_samples=500, seed=3, paradigm=paradigm)
        dr.to_output()


@pytest.mark.parametrize("name", ["fastgcn", "layer"])
def test_collective_many_explicit_samples(name):
    """Collective apps over more than 8,192 caller-given samples (the roots'
    offsets read back exceed the 64 KB staging block of nd_d2h): the rows
    equal those of the two halves run separately."""
    from dataclasses import dataclass

    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph

    @dataclass
    class S:
        id: int
        roots: tuple

    dg = DeviceGraph.rmat(12, 8, seed=3, undirected=True, weighted=False)
    rng = np.random.default_rng(5)
    samples = [S(i, (int(rng.integers(0, dg.n_vertices)),)) for i in range(9000)]
    app = make_app(name)

    def rows(ss):
        dr = run_device(app, dg, ss, seed=9, paradigm="tp")
        off, ids = dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)
        dr.close()
        return [ids[off[i]:off[i + 1]] for i in range(len(off) - 1)]

    whole = rows(samples)
    halves = rows(samples[:4500]) + rows(samples[4500:])
    assert len(whole) == len(halves) == 9000
    assert all(np.array_equal(a, b) for a, b in zip(whole, halves))

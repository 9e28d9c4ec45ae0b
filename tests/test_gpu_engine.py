"""End-to-end parity of the device engine (tp_run / sp_run through the
C-ABI) against the reference's golden hashes and the C oracle."""

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import golden, golden_graph, oracle_run, recorded_equal, sha16, texts

pytestmark = pytest.mark.gpu

WALKS = ("deepwalk", "ppr", "node2vec", "multirw")


def _cases(apps):
    return [m for m in golden("runs.json") if m["app"] in apps]


def _device_run(meta, paradigm):
    from paper_2009_06693_b200 import EngineConfig, make_app, make_samples, sp_run, tp_run
    from paper_2009_06693_b200.graph import DeviceGraph
    g = golden_graph(meta["graph"])
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    app = make_app(meta["app"], **meta["params"])
    samples = make_samples(app, g, meta["n_samples"], meta["seed"])
    run = tp_run if paradigm == "tp" else sp_run
    return run(app, dg, samples, EngineConfig(seed=meta["seed"]))


@pytest.mark.parametrize("paradigm", ["tp", "sp"])
@pytest.mark.parametrize("meta", _cases(WALKS), ids=lambda m: f"{m['idx']}-{m['app']}-{m['graph']}")
def test_walk_runs_match_reference(meta, paradigm):
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
    ("node2vec", {}, True), ("node2vec", {}, False), ("multirw", {"roots_per_sample": 8}, False)])
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
    for par in ("tp", "sp"):
        dr = run_device(a, dg, n_samples=n, seed=9, paradigm=par)
        out = dr.to_output()
        off, ids = out.final_csr()
        roff, rids = ref.final_csr()
        assert np.array_equal(off, roff) and np.array_equal(ids, rids), par
        assert out.n_steps == ref.n_steps
        if par == "tp":
            st = dr.stats()
            got = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in st.timings])
            assert np.array_equal(got.reshape(-1, 3), ref.stats[:, :3])
            assert st.adjacency_fetches == int(ref.stats[:, 3].sum())
        dr.close()

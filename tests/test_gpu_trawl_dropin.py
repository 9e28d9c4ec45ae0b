"""Drop-in on the GPU box: the reference package itself (trawl, installed into
baseline/_ref, which travels with the repo) builds the graph, the apps and
the samples; the same objects go through trawl's own tp_run/sp_run on the
host and through this package's tp_run/sp_run on the device, and every
final row, per-step row and recorded edge is identical (the engine entry of
SURVEY §8(b): transit_parallel.py:249-257, sample_parallel.py:102-110)."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def trawl():
    if not os.path.isdir(os.path.join(REF, "trawl")):
        pytest.skip("baseline/_ref (the installed reference) is absent")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import trawl as T
    from trawl import apps, synth
    from trawl.engine import driver, sample_parallel, transit_parallel
    return {"T": T, "apps": apps, "synth": synth, "driver": driver,
            "tp_run": transit_parallel.tp_run, "sp_run": sample_parallel.sp_run}


CASES = [("deepwalk", {"walk_length": 20}), ("ppr", {"termination_probability": 0.1}),
         ("node2vec", {"walk_length": 20}), ("multirw", {}), ("khop", {"fanouts": [5, 3]}),
         ("layer", {}), ("fastgcn", {}), ("mvs", {}), ("clustergcn", {})]


@pytest.mark.parametrize("paradigm", ["tp", "sp"])
@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_reference_objects_same_rows(trawl, name, kw, paradigm):
    import paper_2009_06693_b200 as P
    graph = trawl["synth"].powerlaw_graph(300, attach=4, weighted=True, seed=3)
    app = trawl["apps"].make_app(name, **kw)
    samples = trawl["driver"].make_samples(app, graph, 40, 11)
    cfg = trawl["driver"].EngineConfig(seed=11)
    ref = trawl[paradigm + "_run"](app, graph, samples, cfg)
    samples = trawl["driver"].make_samples(app, graph, 40, 11)
    ours = (P.tp_run if paradigm == "tp" else P.sp_run)(app, graph, samples, cfg)
    rf, of = ref.final_rows(), ours.final_rows()
    assert len(rf) == len(of)
    for a, b in zip(rf, of):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    for st in range(max(len(s.step_vertices) for s in ref.samples) if ref.samples else 0):
        for a, b in zip(ref.step_rows(st), ours.step_rows(st)):
            assert np.array_equal(np.asarray(a), np.asarray(b))
    for rs, os_ in zip(ref.samples, ours.samples):
        assert len(rs.recorded_edges) == len(os_.recorded_edges)
        for (t0, v0), (t1, v1) in zip(rs.recorded_edges, os_.recorded_edges):
            assert np.array_equal(np.asarray(t0), np.asarray(t1))
            assert np.array_equal(np.asarray(v0), np.asarray(v1))


@pytest.mark.parametrize("paradigm", ["tp", "sp"])
@pytest.mark.parametrize("name,kw", CASES[:5], ids=[c[0] for c in CASES[:5]])
def test_kernel_backend_seam(trawl, name, kw, paradigm, monkeypatch):
    """Level 1 of the boundary (kernels/__init__.py:29-44): trawl's own
    engines with this package's device kernels bound in place of its
    compiled backend (individual_batch; segmented_prefix_sum / segment_max
    for the graph) give the rows of trawl with its own kernels."""
    from paper_2009_06693_b200 import kernels as K
    from trawl.engine import chain, sample_parallel, transit_parallel
    import trawl.graph as TG
    graph = trawl["synth"].powerlaw_graph(300, attach=4, weighted=True, seed=5)
    app = trawl["apps"].make_app(name, **kw)
    cfg = trawl["driver"].EngineConfig(seed=13)
    run = trawl[paradigm + "_run"]
    ref = run(app, graph, trawl["driver"].make_samples(app, graph, 40, 13), cfg)
    calls = []

    def device_batch(*a, **k):  # the device kernel, counted
        calls.append(1)
        return K.individual_batch(*a, **k)

    for mod in (chain, sample_parallel, transit_parallel):
        monkeypatch.setattr(mod, "individual_batch", device_batch)
    monkeypatch.setattr(TG, "segmented_prefix_sum", K.segmented_prefix_sum)
    monkeypatch.setattr(TG, "segment_max", K.segment_max)
    graph2 = trawl["synth"].powerlaw_graph(300, attach=4, weighted=True, seed=5)
    assert np.array_equal(graph2.per_vertex_weight_prefix, graph.per_vertex_weight_prefix)
    ours = run(app, graph2, trawl["driver"].make_samples(app, graph2, 40, 13), cfg)
    assert calls, "trawl's engine did not reach the bound device kernel"
    for a, b in zip(ref.final_rows(), ours.final_rows()):
        assert np.array_equal(np.asarray(a), np.asarray(b))

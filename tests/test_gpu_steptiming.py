"""Per-step build / sample timings (RunStats.timings, StepTiming of
driver.py:42-48, filled per step by transit_parallel.py:204-228) from CUDA
events on the run's stream, under EngineConfig(step_timing=True) or the
engine.profiling() context; outputs are unchanged by the timing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 7


@pytest.fixture(scope="module")
def graph():
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(14, 16, seed=2, weighted=True)
    yield dg
    dg.close()


def _final(out):
    off, ids = out.final_csr()
    return np.asarray(off), np.asarray(ids)


@pytest.mark.parametrize("name,kw,engine", [
    ("khop", {"fanouts": [25, 10]}, "tp"),      # fixed layout, hub-bucket TP
    ("khop", {"fanouts": [25, 10]}, "sp"),      # fixed layout, SP
    ("deepwalk", {}, "tp"),                     # TP hub walk engine (first steps)
    ("fastgcn", {}, "tp"),                      # collective step loop
    ("mvs", {}, "sp"),
])
def test_step_times_recorded(graph, name, kw, engine, monkeypatch):
    from paper_2009_06693_b200 import EngineConfig, make_app, sp_run, tp_run
    monkeypatch.setenv("ND_TP_TAIL", "0")  # every walk step in the hub engine (no walker-major tail)
    from paper_2009_06693_b200.engine import make_samples
    run = tp_run if engine == "tp" else sp_run
    app = make_app(name, **kw)
    n = 20_000 if name == "deepwalk" else 512
    samples = make_samples(app, graph, n, SEED)
    plain = run(app, graph, samples, EngineConfig(seed=SEED))
    timed = run(app, graph, samples, EngineConfig(seed=SEED, step_timing=True))
    po, pi = _final(plain)
    to, ti = _final(timed)
    assert np.array_equal(po, to) and np.array_equal(pi, ti)
    st = timed.stats
    assert st.n_steps >= 1
    first = st.timings[0]
    assert first.sample_s > 0.0 and first.build_s >= 0.0
    assert all(t.sample_s > 0.0 for t in st.timings)  # every step is timed
    assert st.sample_total_s > 0.0
    assert all(t.sample_s == 0.0 for t in plain.stats.timings)


def test_unique_step_loop_times(graph):
    """k-hop with unique() steps runs the generic step loop."""
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import profiling, run_device
    app = make_app("khop", fanouts=[10, 5])
    app.unique = lambda step: True
    with profiling():
        dr = run_device(app, graph, n_samples=256, seed=SEED, paradigm="tp")
    assert len(dr.step_ms) == dr.n_steps >= 1
    assert all(s > 0.0 for _, s in dr.step_ms)
    rs = dr.stats()
    assert [t.sample_s for t in rs.timings] == [s / 1e3 for _, s in dr.step_ms]
    dr.close()

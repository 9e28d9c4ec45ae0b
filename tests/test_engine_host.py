"""Host-side engine API (CPU): the contracts the reference's own tests rely on.

* ``make_samples`` returns a finite sequence: ``list()``, iteration and ``in``
  terminate (the reference returns a list, driver.py:238-250; its tests
  iterate it, test_apps.py:175, test_engines.py:57-60).
* ``describe()`` maps the reference's real ``trawl.make_app`` objects onto the
  same device plan as this package's mirror apps, for every bundled app
  (apps.py:389-413; the engine seam of INTEGRATION.md §2).  Skipped when
  /root/reference is absent (the GPU box).
* a multi-worker concatenation keeps recorded edges step-major, as the
  reference's ``multi_worker_run`` (bench.py:123-153) does.
"""

import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"


def test_make_samples_is_a_finite_sequence():
    from paper_2009_06693_b200 import make_app, make_samples
    from paper_2009_06693_b200.synth import cycle_graph
    g = cycle_graph(50, weighted=True, seed=2)
    app = make_app("deepwalk")
    samples = make_samples(app, g, 3, seed=1)
    got = [s.id for s in samples]
    assert got == [0, 1, 2]
    assert len(list(samples)) == 3
    assert samples[-1].id == 2
    with pytest.raises(IndexError):
        samples[3]
    with pytest.raises(IndexError):
        samples[-4]
    sub = samples[1:3]
    assert [s.id for s in sub] == [1, 2]
    # roots come from the app's keyed initialiser (apps.py:83-103)
    assert all(len(s.roots) == 1 and 0 <= s.roots[0] < 50 for s in samples)


def _trawl():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference sources absent")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import trawl  # noqa: F401
    from trawl import apps as A
    return A


CASES = [
    ("deepwalk", {}), ("deepwalk", {"walk_length": 17}),
    ("ppr", {}), ("ppr", {"termination_probability": 0.05}),
    ("node2vec", {}), ("node2vec", {"p": 0.5, "q": 4.0, "factor_convention": "direct"}),
    ("multirw", {}), ("khop", {}), ("khop", {"fanouts": [5, 3, 2]}),
    ("layer", {}), ("fastgcn", {}), ("ladies", {"distribution": "degree_sq"}),
    ("mvs", {}), ("clustergcn", {}),
]


def _plan_tuple(p):
    return (p.kind, p.name, p.code, tuple(np.asarray(p.kparams, float).tolist()), p.steps, p.R,
            tuple(p.fanouts), p.ckind, p.step_size, p.max_size, p.distribution, p.cps, p.nc,
            None if p.unique is None else tuple(p.unique.tolist()), p.roots_kind)


@pytest.mark.parametrize("name,kw", CASES, ids=lambda x: str(x))
def test_reference_apps_map_to_the_same_device_plan(name, kw):
    A = _trawl()
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import _describe
    try:
        ref_app = A.make_app(name, **kw)
    except TypeError:
        pytest.skip(f"reference make_app({name}) has no parameter in {kw}")
    ours = make_app(name, **kw)
    pr, po = _describe(ref_app), _describe(ours)
    assert _plan_tuple(pr) == _plan_tuple(po)
    assert pr.roots_kind == "keyed"  # the device draws the reference's keyed roots itself


def test_reference_samples_give_the_same_sample_spec():
    """Reference make_samples -> Sample objects with host roots: the ABI spec
    (contiguous ids, roots array) equals the keyed-root spec's roots."""
    A = _trawl()
    from trawl.engine.driver import make_samples as ref_make_samples
    from trawl.synth import powerlaw_graph
    from paper_2009_06693_b200.engine import _describe, _sample_spec
    g = powerlaw_graph(300, attach=3, weighted=True, seed=0)
    app = A.make_app("khop")
    plan = _describe(app)
    samples = ref_make_samples(app, g, 20, seed=5)
    lo, n, roots, off = _sample_spec(samples, plan, 5)
    assert (lo, n) == (0, 20)
    assert np.array_equal(off, np.arange(21))
    exp = np.concatenate([s.roots for s in samples])
    assert np.array_equal(roots, exp)


def test_multi_worker_concat_keeps_recorded_edges():
    from paper_2009_06693_b200.engine import RunStats
    from paper_2009_06693_b200.output import SampleSetOutput
    from paper_2009_06693_b200.runner import _concat

    def part(ids, cnt, rec_counts, rec_t, rec_v):
        n = len(ids)
        return SampleSetOutput(np.asarray(ids), np.arange(n + 1), np.asarray(ids) * 10,
                               len(cnt), step_counts=np.asarray(cnt, np.int64),
                               step_vals=np.arange(int(np.sum(cnt)), dtype=np.int64),
                               rec_counts=np.asarray(rec_counts, np.int64),
                               rec_t=np.asarray(rec_t, np.int64), rec_v=np.asarray(rec_v, np.int64),
                               stats=RunStats(paradigm="tp", n_samples=n))

    # worker 0: samples 0,1; worker 1: sample 2; two steps each
    a = part([0, 1], [[1, 1], [1, 0]], [[1, 2], [0, 1]], [10, 11, 12, 13], [20, 21, 22, 23])
    b = part([2], [[1], [1]], [[2], [1]], [30, 31, 32], [40, 41, 42])
    out = _concat([a, b], None, RunStats(paradigm="tp", n_samples=3))
    assert out.rec_counts.tolist() == [[1, 2, 2], [0, 1, 1]]
    # step-major: step 0 of a, step 0 of b, step 1 of a, step 1 of b
    assert out.rec_t.tolist() == [10, 11, 12, 30, 31, 13, 32]
    s = out.samples
    assert [len(x.recorded_edges) for x in s] == [2, 2, 2]
    assert s[2].recorded_edges[0][0].tolist() == [30, 31]
    assert s[1].recorded_edges[1][1].tolist() == [23]

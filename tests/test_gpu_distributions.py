"""Distributional checks on device output (the north star's validity and
chi-square tests; the reference's tests/test_acceptance.py:119-170 and
tests/test_apps.py pattern).  Parity with the oracle is already bit-exact;
these pin that the keyed RNG feeds the right distributions at scale.

Graph: every vertex has the same ten out-neighbours 0..9 with weights 1..10,
so every weighted pick follows w/55 and every uniform pick 1/10."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

V, K = 1000, 10


def _graph():
    from paper_2009_06693_b200.graph import DeviceGraph
    row = np.arange(V + 1, dtype=np.int64) * K
    col = np.tile(np.arange(K, dtype=np.int64), V)
    w = np.tile(np.arange(1, K + 1, dtype=np.float64), V)
    return DeviceGraph.from_arrays(row, col, w)


def _chi2_p(counts, probs):
    from scipy.stats import chisquare
    counts = np.asarray(counts, dtype=np.float64)
    exp = np.asarray(probs, dtype=np.float64) * counts.sum()
    return chisquare(counts, exp).pvalue


def test_deepwalk_weighted_picks_and_khop_uniform_picks():
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    g = _graph()
    for par in ("sp", "tp"):
        dr = run_device(make_app("deepwalk", walk_length=20), g, n_samples=50_000, seed=3, paradigm=par)
        off, ids = dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)
        mask = np.ones(len(ids), dtype=bool)
        mask[off[:-1]] = False  # drop the roots: every other value is a weighted pick
        counts = np.bincount(ids[mask], minlength=K)[:K]
        assert counts.sum() == 50_000 * 20
        assert _chi2_p(counts, np.arange(1, K + 1) / 55.0) > 1e-3, (par, counts)
        dr.close()
    dr = run_device(make_app("khop"), g, n_samples=20_000, seed=5, paradigm="sp")
    vals = dr.host(_lib.F_STEP_VALS)
    counts = np.bincount(vals[vals >= 0], minlength=K)[:K]
    assert _chi2_p(counts, np.full(K, 1.0 / K)) > 1e-3, counts
    dr.close()


def test_ppr_lengths_geometric():
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    g = _graph()
    term = 0.2
    dr = run_device(make_app("ppr", termination_probability=term), g, n_samples=200_000, seed=11,
                    paradigm="sp")
    off = dr.host(_lib.F_FINAL_OFF)
    L = np.diff(off) - 1  # values after the root: terminated at step L (no dead ends here)
    kmax = 25
    counts = np.bincount(np.minimum(L, kmax), minlength=kmax + 1)
    probs = np.array([(1 - term) ** k * term for k in range(kmax)] + [(1 - term) ** kmax])
    assert _chi2_p(counts, probs) > 1e-3, counts
    assert abs(L.mean() - (1 - term) / term) < 0.05
    dr.close()


def test_node2vec_second_order_transitions():
    """From v = 1 having come from t = 0: neighbours 0 (return, 1/p), 2
    (adjacent to t, 1) and 3 (far, 1/q) with weights 1, 2, 3; p = 2, q = 0.5
    (reciprocal convention) gives P ∝ (0.5, 2, 6).  Walks rooted at 0 whose
    first step went to 1 are counted (tests/test_apps.py brute-force pattern)."""
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    src = [0, 0, 1, 1, 1, 2, 3, 4]
    dst = [1, 2, 0, 2, 3, 1, 4, 0]
    w = [1.0, 1.0, 1.0, 2.0, 3.0, 1.0, 1.0, 1.0]
    g = DeviceGraph.from_edges(np.array(src), np.array(dst), np.array(w), 5)
    for par in ("sp", "tp"):
        dr = run_device(make_app("node2vec", p=2.0, q=0.5, walk_length=2), g, n_samples=500_000,
                        seed=17, paradigm=par)
        off, ids = dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)
        rows = np.diff(off) == 3
        start = off[:-1][rows]
        r0, r1, r2 = ids[start], ids[start + 1], ids[start + 2]
        sel = (r0 == 0) & (r1 == 1)
        counts = np.bincount(r2[sel], minlength=4)[[0, 2, 3]]
        assert counts.sum() > 20_000
        assert _chi2_p(counts, np.array([0.5, 2.0, 6.0]) / 8.5) > 1e-3, (par, counts)
        dr.close()

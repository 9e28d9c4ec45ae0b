"""The transit-parallel walk engine's hub tiers (csrc/nd_walk_hub.cuh).

Walkers released from a few roots on a low-degree graph crowd onto the same
transits, so every step has hubs whose rows are small enough to stage in
shared memory: the thread-block tier (> 256 members), the warp tier (32..256
members) and, on RMAT graphs, the grid tier.  The rows must equal the
walker-major SP engine's, the per-step class statistics the sort-based TP
engine's (itself pinned to the reference's groups, test_gpu_engine.py), and a
sample of the rows the C oracle's (transit_parallel.py:185-230,
chain.py:64-179)."""

import os
from dataclasses import dataclass

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

APPS = (("deepwalk", {}), ("node2vec", {"p": 2.0, "q": 0.5}),
        ("ppr", {"termination_probability": 0.02}))


@dataclass
class _S:
    id: int
    roots: tuple


def _graph(unit):
    from paper_2009_06693_b200.graph import DeviceGraph
    V = 4096
    rng = np.random.default_rng(11)
    src = np.repeat(np.arange(V, dtype=np.int64), 7)
    off = np.tile(np.array([1, 2, 3, 5, 8, 13, 0], dtype=np.int64), V)
    dst = (src + off) % V
    dst[6::7] = (src[6::7] * 7 + 3) % V
    w = np.ones(len(src)) if unit else rng.uniform(1.0, 5.0, len(src))
    # a few vertices without out-edges end walks
    keep = ~np.isin(src, np.arange(0, V, 97))
    return DeviceGraph.from_edges(src[keep], dst[keep], w[keep], V)


def _samples(n, n_roots=64):
    roots = (np.arange(n_roots) * 61 + 5) % 4096
    return [_S(i, (int(roots[i % n_roots]),)) for i in range(n)]


def _run(app, dg, samples, paradigm, env, monkeypatch):
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200 import _lib
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    dr = run_device(app, dg, samples, seed=3, paradigm=paradigm)
    out = {f: dr.host(f) for f in (_lib.F_FINAL_OFF, _lib.F_FINAL_IDS32, _lib.F_CHAIN_LEN,
                                    _lib.F_STATS)}
    out["counters"] = dict(dr.counters)
    out["steps"] = dr.n_steps
    dr.close()
    for k in env:
        monkeypatch.delenv(k)
    return out


@pytest.mark.parametrize("unit", [False, True], ids=["weighted", "unit"])
@pytest.mark.parametrize("name,kw", APPS, ids=[a for a, _ in APPS])
def test_staged_tiers_match_sp_and_sort_engine(name, kw, unit, monkeypatch):
    from paper_2009_06693_b200 import _lib, make_app
    dg = _graph(unit)
    app = make_app(name, **kw)
    samples = _samples(200_000)
    sp = _run(app, dg, samples, "sp", {}, monkeypatch)
    tp = _run(app, dg, samples, "tp", {"ND_TP_TAIL": "0"}, monkeypatch)
    srt = _run(app, dg, samples, "tp", {"ND_TP_TAIL": "0", "ND_TP_ENGINE": "sort"}, monkeypatch)
    for f in (_lib.F_FINAL_OFF, _lib.F_FINAL_IDS32, _lib.F_CHAIN_LEN):
        assert np.array_equal(sp[f], tp[f]), f
    assert np.array_equal(tp[_lib.F_STATS], srt[_lib.F_STATS])
    assert sp["steps"] == tp["steps"] == srt["steps"]
    st = tp[_lib.F_STATS].reshape(-1, 4)
    assert st[:, 1].sum() > 0 and st[:, 2].sum() > 0  # medium and large groups occur
    c = tp["counters"]
    assert c["tp_staged"] > 0, "no hub member was stepped from a staged row"
    assert c["tp_inplace"] > 0
    # every walker-step ran in exactly one tier
    steps_taken = int(tp[_lib.F_CHAIN_LEN].sum())
    assert c["tp_staged"] + c["tp_inplace"] == steps_taken


@pytest.mark.parametrize("name,kw", APPS, ids=[a for a, _ in APPS])
def test_staged_tiers_match_oracle(name, kw, monkeypatch):
    from paper_2009_06693_b200 import _lib, make_app
    dg = _graph(False)
    hg = dg.to_host()
    og = O.OGraph(hg.n_vertices, hg.row_offsets, hg.col_indices, hg.weights,
                  hg.per_vertex_weight_prefix, hg.per_vertex_max_weight, np.arange(hg.n_vertices))
    app = make_app(name, **kw)
    n = 20_000
    samples = _samples(n)
    tp = _run(app, dg, samples, "tp", {"ND_TP_TAIL": "0"}, monkeypatch)
    assert tp["counters"]["tp_staged"] > 0
    roots = np.array([s.roots for s in samples], dtype=np.int64)
    code = {"deepwalk": 0, "ppr": 1, "node2vec": 2}[name]
    kp = {"deepwalk": [], "ppr": [0.02], "node2vec": [2.0, 0.5, 0.0]}[name]
    ref = O.run_chain(og, code, kp, roots, 3, None if name == "ppr" else 100)
    starts = np.concatenate([[0], np.cumsum(ref["chain_len"])])
    exp = []
    for i in range(n):
        vals = ref["chain_vals"][starts[i]:starts[i + 1]]
        exp.append(np.concatenate([roots[i], vals[vals >= 0]]))
    exp = np.concatenate(exp)
    assert np.array_equal(tp[_lib.F_FINAL_IDS32].astype(np.int64), exp)
    assert np.array_equal(tp[_lib.F_CHAIN_LEN], ref["chain_len"])


@pytest.mark.parametrize("kmulti", ["3", "4", "8"])
@pytest.mark.parametrize("unit", [False, True], ids=["weighted", "unit"])
@pytest.mark.parametrize("name,kw", APPS, ids=[a for a, _ in APPS])
def test_multi_step_launches_match(name, kw, unit, kmulti, monkeypatch):
    """Staged tiers off (ND_TW_STAGE=0): K steps per launch (k_tw_multi,
    counts in per-step arrays, walker state in registers between steps) give
    the one-step-per-launch engine's rows, step counts and per-step class
    statistics, and the sort engine's statistics."""
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(14, 16, seed=4, weighted=not unit) if kmulti != "3" else _graph(unit)
    app = make_app(name, **kw)
    samples = _samples(60_000, n_roots=4096 if kmulti != "3" else 64)
    env = {"ND_TP_TAIL": "0", "ND_TW_STAGE": "0"}
    one = _run(app, dg, samples, "tp", {**env, "ND_TW_MULTI": "1"}, monkeypatch)
    mul = _run(app, dg, samples, "tp", {**env, "ND_TW_MULTI": kmulti}, monkeypatch)
    srt = _run(app, dg, samples, "tp", {"ND_TP_TAIL": "0", "ND_TP_ENGINE": "sort"}, monkeypatch)
    sp = _run(app, dg, samples, "sp", {}, monkeypatch)
    for f in (_lib.F_FINAL_OFF, _lib.F_FINAL_IDS32, _lib.F_CHAIN_LEN):
        assert np.array_equal(one[f], mul[f]), f
        assert np.array_equal(sp[f], mul[f]), f
    assert np.array_equal(one[_lib.F_STATS], mul[_lib.F_STATS])
    assert np.array_equal(srt[_lib.F_STATS], mul[_lib.F_STATS])
    assert one["steps"] == mul["steps"] == sp["steps"]
    c = mul["counters"]
    assert c["tp_staged"] == 0
    assert c["tp_inplace"] == int(mul[_lib.F_CHAIN_LEN].sum())
    assert c["slot_bytes"] == one["counters"]["slot_bytes"]  # the §8(d) byte model is per step

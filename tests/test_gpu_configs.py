"""Full-row parity on every BASELINE.json configuration,
device vs the C oracle, value for value.

* C1: the whole job (DeepWalk, 56,944 walkers x 100 on the reference's own
  powerlaw(56944, attach 7) graph), SP and TP (class kernels and tail).
* C2: node2vec and PPR on the keyed RMAT-22 graph (69M weighted edges), a
  65,536-walker prefix of the bench job, SP and TP with every step through
  the class kernels; the bench line compares the whole 8.4M-walker job.
* C3: k-hop (25, 10) on RMAT-18 (114.6M directed unit edges), a 16,384-root
  prefix of the 233,472-root job, SP and TP.
* C4: FastGCN / LADIES (deg^2) / MVS / ClusterGCN on RMAT-22 (117.2M
  directed unit edges): sampled rows and recorded edges of a prefix.
* C5: the 1B-edge RMAT-26 graph: DeepWalk walkers and k-hop roots at the
  start of the job and inside the rank-7-of-8 shard, against the oracle on
  the rows the runs visit (tests/helpers.oracle_subgraph).

References: chain.py:64-179 (walks), driver.py:203-235 + transit_parallel.py
:185-230 (k-hop), collective.py:39-141 (collective), bench.py:123-153
(sharding by sample id).
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import expected_walk_rows, oracle_full_graph, oracle_subgraph

pytestmark = pytest.mark.gpu

CORES = len(os.sched_getaffinity(0))
SEED = 7


def _rows(dr):
    from paper_2009_06693_b200 import _lib
    off, ids = dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)
    return off, ids


def _walk_check(dg, og, app_name, kw, code, kp, steps, n, lo, paradigms, monkeypatch):
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    roots = O.uniform_roots(dg.n_vertices, 1, SEED, lo, n)
    r = O.run_chain(og, code, kp, roots, SEED, steps, paradigm="sp", n_threads=CORES, sample_lo=lo)
    e_off, e_ids = expected_walk_rows(r["roots"], r)
    app = make_app(app_name, **kw)
    for par, tail in paradigms:
        if tail is not None:
            monkeypatch.setenv("ND_TP_TAIL", tail)
        else:
            monkeypatch.delenv("ND_TP_TAIL", raising=False)
        dr = run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm=par)
        off, ids = _rows(dr)
        dr.close()
        assert np.array_equal(off, e_off), (app_name, par, tail)
        assert np.array_equal(ids, e_ids), (app_name, par, tail)
    return int(e_off[-1])


def test_c1_full_job():
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.synth import powerlaw_graph
    g = powerlaw_graph(56944, attach=7, weighted=True, seed=0)
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    og = oracle_full_graph(dg)
    N = g.n_vertices
    roots = O.uniform_roots(N, 1, SEED, 0, N)
    r = O.run_chain(og, 0, [], roots, SEED, 100, paradigm="sp", n_threads=CORES)
    e_off, e_ids = expected_walk_rows(r["roots"], r)
    assert e_off[-1] == N + 5_694_400  # no dead ends
    for par, tail in (("sp", None), ("tp", None), ("tp", "0")):
        if tail is not None:
            os.environ["ND_TP_TAIL"] = tail
        try:
            dr = run_device(make_app("deepwalk"), dg, n_samples=N, seed=SEED, paradigm=par)
        finally:
            os.environ.pop("ND_TP_TAIL", None)
        off, ids = _rows(dr)
        dr.close()
        assert np.array_equal(off, e_off), (par, tail)
        assert np.array_equal(ids, e_ids), (par, tail)
    dg.close()


@pytest.fixture(scope="module")
def c2_graph():
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
    og = oracle_full_graph(dg)
    yield dg, og
    dg.close()


@pytest.mark.parametrize("app_name,kw,code,kp,steps", [
    ("node2vec", {"p": 2.0, "q": 0.5}, 2, [2.0, 0.5, 0.0], 100),
    ("ppr", {"termination_probability": 0.01}, 1, [0.01], None),
])
def test_c2_prefix(c2_graph, app_name, kw, code, kp, steps, monkeypatch):
    dg, og = c2_graph
    # SP (the bench kernel), TP with every step in the class kernels, TP with
    # the class kernels down to 4,096 walkers and the tail after
    _walk_check(dg, og, app_name, kw, code, kp, steps, 1 << 16, 0,
                [("sp", None), ("tp", "0"), ("tp", "4096")], monkeypatch)


def test_c2_shard_prefix(c2_graph, monkeypatch):
    """A block of sample ids deep inside the job (the last rank's shard of a
    2-GPU strong split): keyed roots and draws make it equal the oracle."""
    dg, og = c2_graph
    lo = (1 << 22) - (1 << 14)
    _walk_check(dg, og, "node2vec", {"p": 2.0, "q": 0.5}, 2, [2.0, 0.5, 0.0], 100, 1 << 14, lo,
                [("sp", None), ("tp", "0")], monkeypatch)


def _khop_final(roots, ref):
    """Expected final rows of a run-loop result: roots, then the non-NULL
    values of every step in (step, sample) order."""
    n, R = roots.shape
    cnt, vals = ref["step_counts"], ref["vals"]
    rows = [list(roots[i]) for i in range(n)]
    pos = 0
    for s in range(cnt.shape[0]):
        for i in range(n):
            c = int(cnt[s, i])
            v = vals[pos:pos + c]
            rows[i].extend(v[v >= 0].tolist())
            pos += c
    off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    return off, np.asarray([x for r in rows for x in r], dtype=np.int64)


def _khop_check(dg, og, n, lo, paradigms):
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    roots = list(O.uniform_roots(dg.n_vertices, 1, SEED, lo, n))
    ref = O.run_individual(og, 3, [], [25, 10], roots, SEED, 2, paradigm="tp", sample_lo=lo)
    app = make_app("khop", fanouts=[25, 10])
    for par in paradigms:
        dr = run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm=par)
        out = dr.to_output()
        dr.close()
        assert out.n_steps == ref["n_steps"]
        assert np.array_equal(out.step_counts, ref["step_counts"]), par
        assert np.array_equal(out.step_vals, ref["vals"]), par
        if par == "tp":  # per-step work classes == the reference scheduler's
            st = np.array([[t.groups_small, t.groups_medium, t.groups_large]
                           for t in out.stats.timings])
            assert np.array_equal(st, ref["stats"][:, :3]), st
        # final rows: root, then each step's non-NULL values (output.py:52-69)
        foff, fids = out.final_csr()
        e_off, e_ids = _khop_final(np.asarray(roots).reshape(n, -1), ref)
        assert np.array_equal(foff, e_off), par
        assert np.array_equal(fids, e_ids), par
    return int(ref["vals"].size)


def test_c3_prefix():
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(18, n_edges=57_300_000, seed=0, undirected=True, weighted=False)
    og = oracle_full_graph(dg)
    _khop_check(dg, og, 1 << 14, 0, ("sp", "tp"))
    _khop_check(dg, og, 1 << 12, 1024 * 227, ("sp", "tp"))  # the job's last batch region
    dg.close()


C4_APPS = [("fastgcn", {}, 256), ("ladies", {"distribution": "degree_sq"}, 256),
           ("mvs", {}, 4096), ("clustergcn", {}, 1)]


def test_c4_prefix():
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    from tests.helpers import app_spec
    dg = DeviceGraph.rmat(22, n_edges=58_600_000, seed=0, undirected=True, weighted=False)
    og = oracle_full_graph(dg)
    for name, kw, n in C4_APPS:
        sp = app_spec(name, kw)
        if name == "clustergcn":
            roots = [O.cluster_roots(og.n_vertices, 20, 100, SEED, i) for i in range(n)]
        else:
            roots = list(O.uniform_roots(og.n_vertices, sp["R"], SEED, 0, n))
        ref = O.run_collective(og, sp["kind"], sp["m"], roots, SEED, sp["steps"],
                               distribution=sp.get("distribution", 0))
        for par in ("tp", "sp"):
            dr = run_device(make_app(name, **kw), dg, n_samples=n, seed=SEED, paradigm=par)
            out = dr.to_output()
            dr.close()
            assert np.array_equal(out.step_counts, ref["step_counts"]), (name, par)
            assert np.array_equal(out.step_vals, ref["vals"]), (name, par)
            assert np.array_equal(out.rec_t, ref["rec_t"]), (name, par)
            assert np.array_equal(out.rec_v, ref["rec_v"]), (name, par)
        if name == "clustergcn":
            assert len(ref["rec_t"]) > 1_000_000
    dg.close()


def test_c5_prefix_and_shard():
    """1B-edge RMAT-26: DeepWalk and k-hop rows of the job's first sample ids
    and of the rank-7-of-8 shard (worker_ranges) equal the oracle's."""
    import torch
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.sharding import worker_ranges
    dg = DeviceGraph.rmat(26, n_edges=1 << 30, seed=0, weighted=True)
    assert dg.n_edges == 1 << 30
    N_walk, N_khop = 1 << 23, 1 << 20
    try:
        for lo in (0, worker_ranges(N_walk, 8)[7][0]):
            n = 1 << 12
            dr = run_device(make_app("deepwalk"), dg, n_samples=n, sample_lo=lo, seed=SEED,
                            paradigm="sp")
            off, ids = _rows(dr)
            dr.close()
            og = oracle_subgraph(dg, ids)
            roots = O.uniform_roots(dg.n_vertices, 1, SEED, lo, n)
            r = O.run_chain(og, 0, [], roots, SEED, 100, paradigm="sp", n_threads=CORES,
                            sample_lo=lo)
            e_off, e_ids = expected_walk_rows(r["roots"], r)
            assert np.array_equal(off, e_off), lo
            assert np.array_equal(ids, e_ids), lo
        for lo in (0, worker_ranges(N_khop, 8)[7][0]):
            n = 1 << 10
            dr = run_device(make_app("khop"), dg, n_samples=n, sample_lo=lo, seed=SEED,
                            paradigm="sp")
            out = dr.to_output()
            dr.close()
            roots = O.uniform_roots(dg.n_vertices, 1, SEED, lo, n)
            # transits: the roots and step 0's picks
            s0 = out.step_vals[:int(out.step_counts[0].sum())]
            og = oracle_subgraph(dg, np.concatenate([roots.ravel(), s0]))
            ref = O.run_individual(og, 3, [], [25, 10], list(roots), SEED, 2, paradigm="sp",
                                   sample_lo=lo)
            assert np.array_equal(out.step_counts, ref["step_counts"]), lo
            assert np.array_equal(out.step_vals, ref["vals"]), lo
    finally:
        dg.close()
        torch.cuda.empty_cache()

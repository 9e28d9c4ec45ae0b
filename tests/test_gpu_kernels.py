"""GPU parity of the level-1 kernel backend (C-ABI) against the oracle and the
reference's golden vectors.  Pattern of tests/test_kernels.py:58-88 in the
reference: identical inputs, bit-identical outputs."""

import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import golden, golden_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


@pytest.fixture(scope="module")
def K():
    from paper_2009_06693_b200 import kernels
    return kernels


def test_library_is_native(torch):
    from paper_2009_06693_b200 import _lib
    L = _lib.load()
    assert L.nd_version() == 1
    assert torch.cuda.get_device_capability()[0] >= 10


def test_mod_u64_fuzz(torch):
    """Exact u % d for the fp64-assisted modulo over 2^22 random pairs plus
    edge cases (d = 1, 2^32-1, powers of two, u near 2^64)."""
    from paper_2009_06693_b200 import _lib
    rng = np.random.default_rng(11)
    n = 1 << 22
    u = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    d = np.concatenate([rng.integers(1, 2**32, n // 2, dtype=np.uint64),
                        rng.integers(1, 2**16, n // 4, dtype=np.uint64),
                        (np.uint64(1) << rng.integers(0, 32, n // 4, dtype=np.uint64))])
    edge_u = np.array([0, 1, 2**64 - 1, 2**64 - 2, 2**63, 2**32, 2**32 - 1] * 4, dtype=np.uint64)
    edge_d = np.array([1] * 7 + [2**32 - 1] * 7 + [3] * 7 + [2**31 + 11] * 7, dtype=np.uint64)
    u = np.concatenate([u, edge_u])
    d = np.concatenate([d, edge_d])
    du = torch.from_numpy(u.view(np.int64)).cuda()
    dd = torch.from_numpy(d.view(np.int64)).cuda()
    out = torch.empty_like(du)
    _lib.check(_lib.load().nd_mod_u64(_lib.ptr(du), _lib.ptr(dd), len(u), _lib.ptr(out),
                                      _lib.stream_ptr()))
    got = out.cpu().numpy().view(np.uint64)
    assert np.array_equal(got, u % d)


def test_keyed_u64_known_answers(K):
    kat = golden("kat.json")["key_u64"]
    for key, u, _ in kat:
        seed, sid, step, tix, slot, dom, draw = key
        got = K.keyed_u64(seed, np.array([sid]), step, np.array([tix]), np.array([slot]),
                          domain=dom, draw=draw)
        assert int(got[0]) == int(u), key


@pytest.mark.parametrize("code", [0, 1, 2, 3, 4])
def test_batch_parity_vs_reference(K, code):
    d = golden("batch_parity.npz")
    out = np.empty(len(d[f"c{code}/out"]), dtype=np.int64)
    K.individual_batch(code, d[f"c{code}/params"], d["g/row_offsets"], d["g/col_indices"],
                       d["g/weights"], d["g/prefix"], d["g/max_w"], d[f"c{code}/transits"],
                       d[f"c{code}/t_prev"], d[f"c{code}/sample_ids"], d[f"c{code}/transit_idxs"],
                       d[f"c{code}/slots"], 123, 2, out)
    assert np.array_equal(out, d[f"c{code}/out"])


def test_batch_parity_large_random(K):
    """50k items per app on a 2000-vertex weighted power-law graph vs the C oracle."""
    g = golden_graph("powerlaw:2000|1|7")
    rng = np.random.default_rng(3)
    n = 50_000
    for code, params in [(0, []), (1, [0.2]), (2, [2.0, 0.5, 0.0]), (2, [0.25, 4.0, 1.0]),
                         (3, []), (4, [])]:
        tr = rng.integers(0, g.n_vertices, n)
        tp = np.where(rng.random(n) < 0.8, rng.integers(0, g.n_vertices, n), -1)
        sids, tix, sl = rng.integers(0, 2**40, n), rng.integers(0, 50, n), rng.integers(0, 50, n)
        a = np.empty(n, dtype=np.int64)
        b = np.empty(n, dtype=np.int64)
        args = (code, params, g.row_offsets, g.col_indices, g.weights, g.per_vertex_weight_prefix,
                g.per_vertex_max_weight, tr, tp, sids, tix, sl, 2**63 + 5, 17)
        K.individual_batch(*args, a)
        O.individual_batch(*args, b)
        assert np.array_equal(a, b), code


def test_five_vertex_vectors(K):
    g = O.make_graph([0, 4, 6, 7, 7, 7], [1, 2, 3, 4, 0, 2, 3], [1.5, 2.0, 0.5, 3.0, 1.0, 1.0, 1.0])
    vec = golden("kat.json")["five_vertex"]["batch_seed7_step1"]
    z = np.zeros(8, dtype=np.int64)
    for name, code, params, tprev in [("deepwalk", 0, [], -1), ("ppr", 1, [0.3], -1),
                                      ("khop", 3, [], -1), ("node2vec", 2, [2.0, 0.5, 0.0], 1),
                                      ("node2vec_direct", 2, [2.0, 0.5, 1.0], 1)]:
        out = np.empty(8, dtype=np.int64)
        K.individual_batch(code, params, g.row_offsets, g.col_indices, g.weights,
                           g.per_vertex_weight_prefix, g.per_vertex_max_weight, z,
                           np.full(8, tprev), np.arange(8), z, z, 7, 1, out)
        assert out.tolist() == vec[name], name


def test_prefix_and_max_parity(K):
    for key in ("powerlaw:2000|1|7", "star:300|1|1", "path:300|1|2"):
        g = golden_graph(key)
        assert np.array_equal(K.segmented_prefix_sum(g.weights, g.row_offsets), g.per_vertex_weight_prefix)
        assert np.array_equal(K.segment_max(g.weights, g.row_offsets), g.per_vertex_max_weight)
    # empty segments and a single huge segment
    off = np.array([0, 0, 5, 5, 100005, 100005])
    vals = np.random.default_rng(1).uniform(1, 5, 100005)
    assert np.array_equal(K.segmented_prefix_sum(vals, off), O.segmented_prefix_sum(vals, off))
    assert np.array_equal(K.segment_max(vals, off), O.segment_max(vals, off))


def test_unknown_code_and_stall(K):
    from paper_2009_06693_b200.errors import SamplerStallError
    g = O.make_graph([0, 2, 2, 2], [1, 2], [0.0, 1e-300])
    z = np.zeros(1, dtype=np.int64)
    with pytest.raises(ValueError):
        K.individual_batch(9, [], g.row_offsets, g.col_indices, g.weights,
                           g.per_vertex_weight_prefix, g.per_vertex_max_weight, z, z - 1, z, z, z,
                           0, 0, np.empty(1, dtype=np.int64))
    with pytest.raises(SamplerStallError):
        K.individual_batch(2, [1e300, 1e300, 0.0], g.row_offsets, g.col_indices, g.weights,
                           g.per_vertex_weight_prefix, g.per_vertex_max_weight, z, z + 2, z, z, z,
                           0, 1, np.empty(1, dtype=np.int64))


def test_empty_batch(K):
    g = golden_graph("powerlaw:2000|1|7")
    e = np.empty(0, dtype=np.int64)
    K.individual_batch(0, [], g.row_offsets, g.col_indices, g.weights, g.per_vertex_weight_prefix,
                       g.per_vertex_max_weight, e, e, e, e, e, 1, 0, e)


def test_graph_arrays_upload_once(K):
    """The level-1 seam keeps one device copy per host graph array (the
    reference's Graph is frozen, graph.py:36-39); repeated per-step calls reuse
    it and give the same results."""
    d = golden("batch_parity.npz")
    g = {k: np.ascontiguousarray(d[f"g/{k}"]) for k in ("row_offsets", "col_indices", "weights",
                                                         "prefix", "max_w")}
    K.clear_graph_cache()
    outs = []
    for rep in range(3):
        out = np.empty(len(d["c0/out"]), dtype=np.int64)
        K.individual_batch(0, d["c0/params"], g["row_offsets"], g["col_indices"], g["weights"],
                           g["prefix"], g["max_w"], d["c0/transits"], d["c0/t_prev"],
                           d["c0/sample_ids"], d["c0/transit_idxs"], d["c0/slots"], 123, 2, out)
        outs.append(out)
        if rep == 0:
            cached = {k: v[4].data_ptr() for k, v in K._GRAPH_CACHE.items()}
            assert len(cached) == 5
    assert {k: v[4].data_ptr() for k, v in K._GRAPH_CACHE.items()} == cached
    for o in outs:
        assert np.array_equal(o, d["c0/out"])
    # a different array object is a different graph
    w2 = g["weights"].copy()
    K.individual_batch(0, d["c0/params"], g["row_offsets"], g["col_indices"], w2, g["prefix"],
                       g["max_w"], d["c0/transits"], d["c0/t_prev"], d["c0/sample_ids"],
                       d["c0/transit_idxs"], d["c0/slots"], 123, 2, outs[0])
    assert len(K._GRAPH_CACHE) == 6
    del w2
    assert len(K._GRAPH_CACHE) == 5

"""Pin the C oracle against the reference's own outputs (CPU only).

Every fixture under tests/golden/ was produced by running the reference
(trawl, compiled Cython backend) — see tests/golden/make_golden.py.  The
oracle must reproduce them exactly before it is trusted as the checker for
the CUDA engine.
"""

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import golden, golden_graph, oracle_run, recorded_equal, sha16, texts


def test_key_u64_known_answers():
    for key, u, unif in golden("kat.json")["key_u64"]:
        assert O.key_u64(*key) == int(u), key
        assert O.key_uniform(*key) == unif, key


def test_survey_appendix_c_kats():
    assert O.key_u64(0, 0, 0, 0, 0, 0, 0) == 0xCB34B376670B5E8F
    assert O.key_u64(7, 3, 2, 1, 4, 0, 9) == 0xF7A1658B7BEADE0F
    assert O.key_uniform(7, 3, 2, 1, 4, 0, 9) == 0.9673064675843465
    assert O.key_u64(2**64 - 1, 10**6, 99, 24, 9, 1, 5) == 0x443F7E6ABFF6EED8


def five_vertex():
    return O.make_graph([0, 4, 6, 7, 7, 7], [1, 2, 3, 4, 0, 2, 3],
                        [1.5, 2.0, 0.5, 3.0, 1.0, 1.0, 1.0])


def test_five_vertex_prefix_and_max():
    g = five_vertex()
    kat = golden("kat.json")["five_vertex"]
    assert g.per_vertex_weight_prefix.tolist() == kat["prefix"]
    assert g.per_vertex_max_weight.tolist() == kat["max_w"]


@pytest.mark.parametrize("name,code,params,tprev", [
    ("deepwalk", 0, [], -1), ("ppr", 1, [0.3], -1), ("khop", 3, [], -1),
    ("multirw", 4, [], -1), ("node2vec", 2, [2.0, 0.5, 0.0], 1),
    ("node2vec_direct", 2, [2.0, 0.5, 1.0], 1)])
def test_five_vertex_batch_vectors(name, code, params, tprev):
    g = five_vertex()
    n = 8
    z = np.zeros(n, dtype=np.int64)
    out = np.empty(n, dtype=np.int64)
    O.individual_batch(code, params, g.row_offsets, g.col_indices, g.weights,
                       g.per_vertex_weight_prefix, g.per_vertex_max_weight, z,
                       np.full(n, tprev), np.arange(n), z, z, 7, 1, out)
    assert out.tolist() == golden("kat.json")["five_vertex"]["batch_seed7_step1"][name]


@pytest.mark.parametrize("code", [0, 1, 2, 3, 4])
def test_batch_parity_vs_reference(code):
    d = golden("batch_parity.npz")
    out = np.empty(len(d[f"c{code}/out"]), dtype=np.int64)
    O.individual_batch(code, d[f"c{code}/params"], d["g/row_offsets"], d["g/col_indices"],
                       d["g/weights"], d["g/prefix"], d["g/max_w"], d[f"c{code}/transits"],
                       d[f"c{code}/t_prev"], d[f"c{code}/sample_ids"], d[f"c{code}/transit_idxs"],
                       d[f"c{code}/slots"], 123, 2, out)
    assert np.array_equal(out, d[f"c{code}/out"])


def test_unknown_app_code_raises():
    g = five_vertex()
    z = np.zeros(1, dtype=np.int64)
    with pytest.raises(ValueError):
        O.individual_batch(9, [], g.row_offsets, g.col_indices, g.weights,
                           g.per_vertex_weight_prefix, g.per_vertex_max_weight,
                           z, z - 1, z, z, z, 0, 0, np.empty(1, dtype=np.int64))


def test_node2vec_stall_raises():
    # all weights zero but envelope positive is impossible; use env > 0 with
    # weights 0 on picks: vertex 0 -> 1 (w 0) and 0 -> 2 (w 1); max_w 1;
    # prev t = 2 whose adjacency is empty; q huge -> f_far tiny; p huge.
    g = O.make_graph([0, 2, 2, 2], [1, 2], [0.0, 1e-300])
    z = np.zeros(1, dtype=np.int64)
    with pytest.raises(O.OracleStallError):
        O.individual_batch(2, [1e300, 1e300, 0.0], g.row_offsets, g.col_indices, g.weights,
                           g.per_vertex_weight_prefix, g.per_vertex_max_weight,
                           z, z + 2, z, z, z, 0, 1, np.empty(1, dtype=np.int64))


def _cases():
    return golden("runs.json")


@pytest.mark.parametrize("meta", _cases(), ids=lambda m: f"{m['idx']}-{m['app']}-{m['graph']}-{m['seed']}")
def test_oracle_runs_match_reference(meta):
    g = golden_graph(meta["graph"])
    out = oracle_run(meta, g)
    tf, ts = texts(out)
    assert out.n_steps == meta["n_steps"]
    assert sha16(tf) == meta["hash_final"]
    assert sha16(ts) == meta["hash_per_step"]
    assert out.total_sampled() == meta["total_sampled"]
    rs = golden("runs.npz")
    pre = f"r{meta['idx']}"
    assert recorded_equal(out, rs, pre)
    # transit-parallel group classes per step (StepTiming.groups_*)
    assert np.array_equal(out.stats[:, :3], rs[f"{pre}/groups"])
    assert int(out.stats[:, 3].sum()) == meta["adjacency_fetches"]


def test_oracle_sp_equals_tp_and_threads():
    metas = [m for m in _cases() if m["app"] in ("deepwalk", "ppr", "node2vec", "multirw", "khop")][:12]
    for meta in metas:
        g = golden_graph(meta["graph"])
        ref = texts(oracle_run(meta, g, paradigm="tp"))
        assert texts(oracle_run(meta, g, paradigm="sp")) == ref
        if meta["app"] != "khop":
            assert texts(oracle_run(meta, g, paradigm="tp", n_threads=4)) == ref


@pytest.mark.parametrize("ci", range(5))
def test_schedule_export_matches_reference(ci):
    d = golden("schedule.npz")
    r = O.transit_schedule(d[f"s{ci}/pair_transit"], int(d[f"s{ci}/m"][0]))
    assert np.array_equal(r["order"], d[f"s{ci}/order"])
    assert np.array_equal(np.diff(r["group_start"]), d[f"s{ci}/group_size"])
    assert np.array_equal(r["group_transit"], d[f"s{ci}/group_transit"])
    assert np.array_equal(r["group_class"], d[f"s{ci}/group_class"])
    assert np.array_equal(r["sched_index"], d[f"s{ci}/sched_index"])


@pytest.mark.parametrize("key", ["s9_8_0_1", "s8_4_1_0", "s10_16_0_1"])
def test_csr_build_matches_reference_from_edges(key):
    d = golden("csr_rmat.npz")
    scale, ef, und, wt = (int(x) for x in key[1:].split("_"))
    src, dst, w = O.rmat_edges(scale, (1 << scale) * ef, seed=scale, undirected=bool(und), weighted=bool(wt))
    assert np.array_equal(src, d[f"{key}/src"]) and np.array_equal(dst, d[f"{key}/dst"])
    assert np.array_equal(w, d[f"{key}/w"])
    g = O.from_edges(src, dst, w if wt else None, 1 << scale)
    assert np.array_equal(g.row_offsets, d[f"{key}/row_offsets"])
    assert np.array_equal(g.col_indices, d[f"{key}/col_indices"])
    assert np.array_equal(g.weights, d[f"{key}/weights"])
    assert np.array_equal(g.per_vertex_weight_prefix, d[f"{key}/prefix"])
    assert np.array_equal(g.per_vertex_max_weight, d[f"{key}/max_w"])


def test_worker_ranges_semantics():
    from paper_2009_06693_b200.sharding import worker_ranges
    for k, v in golden("kat.json")["worker_ranges"].items():
        n, w = (int(x) for x in k.split("_"))
        assert [list(r) for r in worker_ranges(n, w)] == v

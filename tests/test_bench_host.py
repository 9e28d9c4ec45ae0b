"""bench.py's host-side checks (CPU): the full-row parity comparison of the
device's final rows with the oracle's chains detects any changed value."""

import numpy as np

import bench
from tests.helpers import expected_walk_rows


def _chain():
    # three walkers: lengths 3 (dies at step 2: NULL), 2 (alive), 1 (dies at step 0)
    return {"chain_len": np.array([3, 2, 1]), "chain_vals": np.array([5, 6, -1, 7, 8, -1])}


def test_rows_equal_chain_exact():
    r = _chain()
    roots = np.array([1, 2, 3])
    off = np.array([0, 3, 6, 7])
    ids = np.array([1, 5, 6, 2, 7, 8, 3])
    assert bench.rows_equal_chain(off, ids, roots, r)
    e_off, e_ids = expected_walk_rows(roots, r)
    assert np.array_equal(e_off, off) and np.array_equal(e_ids, ids)
    for k in range(len(ids)):
        bad = ids.copy()
        bad[k] += 1
        assert not bench.rows_equal_chain(off, bad, roots, r), k
    assert not bench.rows_equal_chain(np.array([0, 3, 5, 7]), ids, roots, r)

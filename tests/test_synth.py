"""The input generators reproduce the reference-built golden graphs."""

import numpy as np
import pytest

from paper_2009_06693_b200.synth import make_synthetic
from tests.helpers import golden


@pytest.mark.parametrize("key", ["cycle:200|0|7", "powerlaw:2000|1|7", "powerlaw:2000|0|3",
                                 "path:300|1|1", "star:300|1|2", "powerlaw:1000|1|5"])
def test_generators_match_reference(key):
    spec, wt, seed = key.split("|")
    g = make_synthetic(spec, weighted=bool(int(wt)), seed=int(seed))
    d = golden("graphs.npz")
    assert np.array_equal(g.row_offsets, d[f"{key}/row_offsets"])
    assert np.array_equal(g.col_indices, d[f"{key}/col_indices"])
    assert np.array_equal(g.weights, d[f"{key}/weights"])


def test_weighted_chunk_plan():
    from paper_2009_06693_b200.streaming import chunk_plan, weighted_plan
    assert weighted_plan(100, (1, 4, 4, 1)) == [(0, 10), (10, 50), (50, 90), (90, 100)]
    assert weighted_plan(0, (1, 2)) == [] and chunk_plan(0, 3) == []
    parts = weighted_plan(12345, (0.5, 5, 5, 5, 1))
    assert parts[0][0] == 0 and parts[-1][1] == 12345
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    with pytest.raises(ValueError):
        weighted_plan(10, (1, 0))

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

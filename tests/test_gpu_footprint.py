"""HBM footprint of a resident graph and the plain-CSR path taken when the
accelerating indexes/records do not fit (nd_index.cu room checks).

Every index (guide tables, hash sets, packed neighbour records, pick lines)
is an accelerator over the reference's own CSR reads (graph.py:78-97,
_ckernels.pyx:65-100): a run that finds no room for one reads the plain CSR
and must return the same rows.  The subprocess below sets the room margin
above any GPU's memory, so every structure is left out.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import expected_walk_rows, oracle_full_graph

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 7
WALKS = (("deepwalk", {}, 0, [], 100), ("node2vec", {"p": 2.0, "q": 0.5}, 2, [2.0, 0.5, 0.0], 100),
         ("ppr", {"termination_probability": 0.01}, 1, [0.01], None))

_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2009_06693_b200 import make_app, _lib
from paper_2009_06693_b200.engine import run_device
from paper_2009_06693_b200.graph import DeviceGraph
dg = DeviceGraph.rmat(14, 16, seed=3, weighted=True)
out = {}
for name, kw in (("deepwalk", {}), ("node2vec", {"p": 2.0, "q": 0.5}),
                 ("ppr", {"termination_probability": 0.01})):
    for par in ("sp", "tp"):
        dr = run_device(make_app(name, **kw), dg, n_samples=8192, seed=7, paradigm=par)
        out[name + "/" + par] = [dr.host(_lib.F_FINAL_OFF).tolist(), dr.host(_lib.F_FINAL_IDS).tolist()]
        dr.close()
out["footprint"] = dg.footprint()
print(json.dumps(out))
"""


def _expected(dg, og, code, kp, steps, n):
    roots = O.uniform_roots(dg.n_vertices, 1, SEED, 0, n)
    r = O.run_chain(og, code, kp, roots, SEED, steps, paradigm="sp", n_threads=4)
    return expected_walk_rows(r["roots"], r)


def test_plain_csr_when_no_room():
    from paper_2009_06693_b200.graph import DeviceGraph
    env = dict(os.environ, ND_INDEX_MARGIN_MB=str(1 << 40))
    p = subprocess.run([sys.executable, "-c", _CHILD, REPO], env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    got = json.loads(p.stdout.strip().splitlines()[-1])
    fp = got["footprint"]
    assert fp["built"] == [] and fp["index_bytes"] == 0
    assert {"vrec", "nbw", "nbp", "guide", "hset", "pick_lines"} <= set(fp["skipped_no_room"])
    dg = DeviceGraph.rmat(14, 16, seed=3, weighted=True)
    og = oracle_full_graph(dg)
    for name, _, code, kp, steps in WALKS:
        e_off, e_ids = _expected(dg, og, code, kp, steps, 8192)
        for par in ("sp", "tp"):
            off, ids = got[f"{name}/{par}"]
            assert np.array_equal(np.asarray(off), e_off), (name, par)
            assert np.array_equal(np.asarray(ids), e_ids), (name, par)
    dg.close()


def test_footprint_reports_built_indexes():
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(12, 16, seed=1, weighted=True)
    fp0 = dg.footprint()
    assert fp0["index_bytes"] == 0 and fp0["built"] == [] and fp0["csr_bytes"] == dg.resident_bytes()
    V, E = dg.n_vertices, dg.n_edges
    assert fp0["csr_bytes"] >= (V + 1) * 8 + E * 4 + 2 * E * 8
    run_device(make_app("node2vec", p=2.0, q=0.5), dg, n_samples=1024, seed=SEED).close()
    fp = dg.footprint()
    assert {"vrec", "nbw", "nbp", "guide", "hset"} <= set(fp["built"])
    assert fp["skipped_no_room"] == []
    assert fp["index_bytes"] == dg.resident_bytes() - fp["csr_bytes"] > 0
    assert fp["prep_ms"] > 0.0
    run_device(make_app("deepwalk"), dg, n_samples=1024, seed=SEED).close()
    assert "pick_lines" in dg.footprint()["built"]
    dg.close()

"""NDSO binary output (output.py:108-142 of the reference) against the bytes
the reference's own write_binary produced for the SURVEY Appendix C runs
(tests/golden/ndso.json, from tests/golden/make_golden_ndso.py): CPU through
the oracle's rows, GPU through the device engine's rows."""

import hashlib
import json
import os

import pytest

from tests.helpers import build_app, golden_graph, oracle_run

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NDSO = {e["idx"]: e for e in json.load(open(os.path.join(GOLD, "ndso.json")))}
RUNS = [m for m in json.load(open(os.path.join(GOLD, "runs.json"))) if m["idx"] in NDSO]


def _digests(out, tmp_path):
    from paper_2009_06693_b200.output import LAYOUT_FINAL, LAYOUT_PER_STEP, write_binary
    d = {}
    for layout in (LAYOUT_FINAL, LAYOUT_PER_STEP):
        p = tmp_path / f"o.{layout}.ndso"
        write_binary(out, layout, str(p))
        d[layout] = hashlib.sha256(p.read_bytes()).hexdigest()
    return d


@pytest.mark.parametrize("meta", RUNS, ids=lambda m: f"{m['idx']}-{m['app']}")
def test_ndso_bytes_match_reference_oracle_rows(meta, tmp_path):
    out = oracle_run(meta, golden_graph(meta["graph"]))
    got = _digests(out, tmp_path)
    exp = NDSO[meta["idx"]]
    assert got["final"] == exp["final"] and got["per-step"] == exp["per-step"]


@pytest.mark.gpu
@pytest.mark.parametrize("meta", RUNS, ids=lambda m: f"{m['idx']}-{m['app']}")
def test_ndso_bytes_match_reference_device_rows(meta, tmp_path):
    from paper_2009_06693_b200 import EngineConfig, make_samples, tp_run
    from paper_2009_06693_b200.graph import DeviceGraph
    g = golden_graph(meta["graph"])
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    app = build_app(meta)
    out = tp_run(app, dg, make_samples(app, g, meta["n_samples"], meta["seed"]),
                 EngineConfig(seed=meta["seed"]))
    got = _digests(out, tmp_path)
    exp = NDSO[meta["idx"]]
    assert got["final"] == exp["final"] and got["per-step"] == exp["per-step"]

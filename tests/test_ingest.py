"""Edge-list ingestion against the reference's own
load_edge_list (graph.py:132-188): golden CSR arrays and errors from
tests/golden/make_golden_ingest.py.

CPU: the host mirror (paper_2009_06693_b200.graph.load_edge_list, whose
per-line rules the device path also uses for the lines it leaves to the
host).  GPU: DeviceGraph.from_edge_list — parse, id compaction and CSR build
on device — bit-exact (weights compared as bit patterns: NaN and -0.0 kept).
"""

import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(GOLD, "ingest.json")))
ARR = np.load(os.path.join(GOLD, "ingest.npz"))


def _write(tmp_path, case):
    p = tmp_path / (case["name"] + ".txt")
    p.write_bytes(ARR[f"{case['name']}/text"].tobytes())
    return str(p)


def _same_graph(case, row, col, w, remap):
    n = case["name"]
    assert np.array_equal(row, ARR[f"{n}/row_offsets"])
    assert np.array_equal(col, ARR[f"{n}/col_indices"])
    ew = np.asarray(ARR[f"{n}/weights"], dtype=np.float64)
    assert np.array_equal(np.asarray(w, np.float64).view(np.int64), ew.view(np.int64))
    assert np.array_equal(remap, ARR[f"{n}/remap"])


def _check(case, load):
    from paper_2009_06693_b200.errors import EmptyGraphError, GraphParseError
    if case["ok"]:
        return load()
    exc = {"GraphParseError": GraphParseError, "EmptyGraphError": EmptyGraphError,
           "OverflowError": OverflowError}[case["error"]]
    with pytest.raises(exc) as err:
        load()
    if case["error"] == "GraphParseError":
        assert err.value.line_no == case["line_no"]
        assert str(err.value) == case["message"]
    return None


@pytest.mark.parametrize("case", META, ids=lambda c: c["name"])
def test_host_parser_matches_reference(case, tmp_path):
    from paper_2009_06693_b200.graph import load_edge_list
    path = _write(tmp_path, case)
    g = _check(case, lambda: load_edge_list(path, **case["kwargs"]))
    if g is not None:
        _same_graph(case, g.row_offsets, g.col_indices, g.weights, g.remap)


@pytest.mark.gpu
@pytest.mark.parametrize("case", META, ids=lambda c: c["name"])
def test_device_ingestion_matches_reference(case, tmp_path):
    from paper_2009_06693_b200.graph import DeviceGraph
    path = _write(tmp_path, case)
    dg = _check(case, lambda: DeviceGraph.from_edge_list(path, **case["kwargs"]))
    if dg is not None:
        h = dg.to_host()
        _same_graph(case, h.row_offsets, h.col_indices, h.weights, h.remap)
        dg.close()


@pytest.mark.gpu
def test_device_cache_roundtrip(tmp_path):
    """NDGR cache (graph.py:191-217) written by the host mirror, loaded to HBM."""
    from paper_2009_06693_b200.graph import DeviceGraph, load_edge_list, save_cache
    case = next(c for c in META if c["name"] == "big_mixed")
    g = load_edge_list(_write(tmp_path, case), **case["kwargs"])
    save_cache(g, str(tmp_path / "g.ndgr"))
    dg = DeviceGraph.from_cache(str(tmp_path / "g.ndgr"))
    h = dg.to_host()
    _same_graph(case, h.row_offsets, h.col_indices, h.weights, h.remap)
    dg.close()


@pytest.mark.gpu
def test_readme_quickstart(tmp_path):
    """The README's usage snippet: ingest on device, sample, read rows."""
    from paper_2009_06693_b200 import EngineConfig, make_app, make_samples, sp_run
    from paper_2009_06693_b200.graph import DeviceGraph
    case = next(c for c in META if c["name"] == "big_mixed")
    g = DeviceGraph.from_edge_list(_write(tmp_path, case), weighted=True)
    app = make_app("node2vec")
    out = sp_run(app, g, make_samples(app, g, 1000, seed=7), EngineConfig(seed=7))
    rows = out.final_rows()
    assert len(rows) == 1000 and all(len(r) >= 1 for r in rows)

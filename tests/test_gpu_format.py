"""Text rows printed on the device (nd_format_rows) equal the reference's
text writer (output.py:72-92 render_text / emit, remap output.py:145-150),
byte for byte: empty rows, remapped labels (including negative and 19-digit
ones), int32 and int64 ids, and a whole engine run in both layouts."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _py_text(sample_ids, off, ids, remap):
    from paper_2009_06693_b200.output import _fmt_rows
    lines = []
    _fmt_rows(sample_ids, off, ids if remap is None else np.asarray(remap)[ids], lines)
    return "".join(line + "\n" for line in lines).encode()


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("with_remap", [False, True])
def test_rows_match_python_writer(dtype, with_remap):
    from paper_2009_06693_b200.output import _device_rows_text
    rng = np.random.default_rng(3)
    n = 5000
    lens = rng.integers(0, 70, n)
    lens[::17] = 0  # empty rows print "<sid>: "
    lens[5] = 1000  # a row longer than many warps' chunks
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    V = 100_000
    ids = rng.integers(0, V, off[-1]).astype(dtype)
    sids = rng.integers(0, 1 << 40, n).astype(np.int64)
    sids[0] = 0
    remap = None
    if with_remap:
        remap = rng.integers(-(1 << 62), 1 << 62, V).astype(np.int64)
        remap[:10] = [0, -1, 9, 10, -10, 99, 100, (1 << 63) - 1, -(1 << 63), 7]
        ids[:10] = np.arange(10)
    got = _device_rows_text(sids, off, ids, remap)
    assert bytes(got) == _py_text(sids, off, ids, remap)


def test_empty_and_single():
    from paper_2009_06693_b200.output import _device_rows_text
    off = np.zeros(4, dtype=np.int64)
    sids = np.array([0, 7, 123456789], dtype=np.int64)
    assert bytes(_device_rows_text(sids, off, np.empty(0, dtype=np.int64), None)) == b"0: \n7: \n123456789: \n"
    off = np.array([0, 1], dtype=np.int64)
    assert bytes(_device_rows_text(np.array([5], dtype=np.int64), off, np.array([42], dtype=np.int32),
                                   None)) == b"5: 42\n"


@pytest.mark.parametrize("name,kw", [("node2vec", {}), ("khop", {"fanouts": [10, 5]})])
def test_engine_output_text_layouts(name, kw, monkeypatch):
    from paper_2009_06693_b200 import EngineConfig, make_app, output as O, sp_run
    from paper_2009_06693_b200.engine import make_samples
    from paper_2009_06693_b200.graph import DeviceGraph
    dg = DeviceGraph.rmat(14, 16, seed=2, weighted=True)
    app = make_app(name, **kw)
    out = sp_run(app, dg, make_samples(app, dg, 4000, 7), EngineConfig(seed=7))
    for layout in (O.LAYOUT_FINAL, O.LAYOUT_PER_STEP):
        monkeypatch.setattr(O, "DEVICE_FORMAT_MIN_IDS", 0)
        dev = O.render_bytes(out, layout)
        monkeypatch.setattr(O, "DEVICE_FORMAT_MIN_IDS", 1 << 62)
        host = O.render_bytes(out, layout)
        assert dev == host
        assert O.render_text(out, layout) == host.decode()

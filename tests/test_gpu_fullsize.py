"""Size-independent properties at BASELINE.json's full C2 size (RMAT scale 22,
68,993,773 weighted edges, node2vec p=2 q=0.5 and PPR 0.01, one walk per
vertex), where the oracle would take too long inside the test suite (bench.py
compares the full job with the oracle on all host cores):

* the SP (walker-major) and TP (transit-parallel, with its tail hand-off)
  engines produce identical rows, element for element;
* every step of every walk follows an edge of the graph;
* a node2vec walk shorter than its length ends at a vertex without out-edges,
  and no walk is longer than the reference allows.
"""

import pytest

pytestmark = pytest.mark.gpu


def _edge_keys(h, torch):
    V = h.n_vertices
    row = torch.from_numpy(h.row_offsets).cuda()
    col = torch.from_numpy(h.col_indices).cuda()
    deg = row[1:] - row[:-1]
    src = torch.repeat_interleave(torch.arange(V, device="cuda"), deg)
    keys, _ = torch.sort(src * V + col.to(torch.int64))
    return keys, deg


def _steps_are_edges(off, ids, keys, V, torch):
    ids = ids.to(torch.int64)
    n = off.numel() - 1
    lens = off[1:] - off[:-1]
    row_of = torch.repeat_interleave(torch.arange(n, device="cuda"), lens)
    same = row_of[1:] == row_of[:-1]  # consecutive entries of one row
    a, b = ids[:-1][same], ids[1:][same]
    q = a * V + b
    pos = torch.searchsorted(keys, q).clamp_(max=keys.numel() - 1)
    return bool((keys[pos] == q).all().item()), int(q.numel())


def test_c2_full_size_properties():
    import torch
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    g = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
    h = g.to_host()
    V = h.n_vertices
    keys, deg = _edge_keys(h, torch)
    for name, kw, max_len in (("node2vec", {"p": 2.0, "q": 0.5}, 101), ("ppr", {"termination_probability": 0.01}, None)):
        app = make_app(name, **kw)
        sp = run_device(app, g, n_samples=V, seed=7, paradigm="sp")
        tp = run_device(app, g, n_samples=V, seed=7, paradigm="tp")
        off, ids = sp.view(_lib.F_FINAL_OFF), sp.view(_lib.F_FINAL_IDS32)
        assert torch.equal(off, tp.view(_lib.F_FINAL_OFF)), name
        assert torch.equal(ids, tp.view(_lib.F_FINAL_IDS32)), name
        ok, n_steps = _steps_are_edges(off, ids, keys, V, torch)
        assert ok and n_steps == sp.total_sampled, name
        lens = off[1:] - off[:-1]
        if max_len is not None:
            assert int(lens.max().item()) <= max_len
            short = lens < max_len
            last = ids[(off[1:] - 1)[short]].to(torch.int64)
            assert bool((deg[last] == 0).all().item()), name
        sp.close()
        tp.close()


def test_c3_c4_full_size_sp_equals_tp():
    """C3 k-hop (25,10) over 233,472 roots of the 114.6M-edge graph and C4
    ClusterGCN over the 117.2M-edge graph: both paradigms, identical rows and
    recorded edges."""
    import torch
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    cases = [((18, 57_300_000), "khop", 233_472, (_lib.F_FINAL_OFF, _lib.F_FINAL_IDS32)),
             ((22, 58_600_000), "clustergcn", 8, (_lib.F_FINAL_OFF, _lib.F_REC_T, _lib.F_REC_V))]
    for (scale, edges), name, n, fields in cases:
        g = DeviceGraph.rmat(scale, n_edges=edges, seed=0, undirected=True, weighted=False)
        sp = run_device(make_app(name), g, n_samples=n, seed=7, paradigm="sp")
        tp = run_device(make_app(name), g, n_samples=n, seed=7, paradigm="tp")
        for f in fields:
            assert torch.equal(sp.view(f), tp.view(f)), (name, f)
        assert sp.total_sampled == tp.total_sampled
        sp.close()
        tp.close()
        g.close()

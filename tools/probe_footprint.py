"""Dev probe: walk rate vs graph footprint (same mean degree, same walker
count), to separate translation reach from per-step instruction latency."""
import json, sys, os, ctypes as C
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app, _lib  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

W = 1 << 22
for scale in (17, 18, 19, 20, 21, 22):
    dg = DeviceGraph.rmat(scale, n_edges=int(16.45 * (1 << scale)), seed=0, weighted=True)
    for app_name in ("deepwalk", "node2vec"):
        app = make_app(app_name)
        dr = run_device(app, dg, n_samples=W, seed=7, paradigm="sp"); dr.close()
        ms = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); dr = run_device(app, dg, n_samples=W, seed=7, paradigm="sp"); e.record()
            torch.cuda.synchronize(); ms.append(s.elapsed_time(e)); tot = dr.total_sampled; dr.close()
        m = sorted(ms)[1]
        print(json.dumps({"scale": scale, "E": dg.n_edges, "bytes": dg.resident_bytes(), "app": app_name,
                          "ms": m, "Gsteps_s": tot / m / 1e6}), flush=True)
    c = C.c_double()
    _lib.load().nd_gather_ceiling(C.c_int64(max(dg.resident_bytes(), 1 << 26)), 4, 32, C.byref(c), None)
    print(json.dumps({"scale": scale, "gather_ceiling_Gs": c.value / 1e9}), flush=True)
    dg.close()

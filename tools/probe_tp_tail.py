"""Dev probe: TP walk time with and without the walker-major tail (C1, C2 apps)."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.synth import powerlaw_graph  # noqa: E402

cases = [("C1 deepwalk", DeviceGraph.from_graph(powerlaw_graph(56944, attach=7, weighted=True, seed=0)),
          make_app("deepwalk"), None)]
g2 = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
cases += [("C2 node2vec", g2, make_app("node2vec", p=2.0, q=0.5), None),
          ("C2 ppr", g2, make_app("ppr", termination_probability=0.01), None)]
for name, g, app, _ in cases:
    for tail in ("0", "131072"):
        os.environ["ND_TP_TAIL"] = tail
        ms = []
        for it in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dr = run_device(app, g, n_samples=g.n_vertices, seed=7, paradigm="tp")
            e.record(); torch.cuda.synchronize()
            ms.append(s.elapsed_time(e))
            if it == 2:
                import hashlib
                from paper_2009_06693_b200 import _lib
                hsh = hashlib.sha1()
                for f in (_lib.F_FINAL_OFF, _lib.F_FINAL_IDS32, _lib.F_STATS, _lib.F_CHAIN_LEN):
                    hsh.update(dr.host(f).tobytes() if hasattr(dr.host(f), "tobytes") else bytes(dr.host(f)))
                tot, steps, dig = dr.total_sampled, dr.n_steps, hsh.hexdigest()[:12]
            dr.close()
        print(f"{name:12s} tail={tail:7s} ms={statistics.median(ms):8.2f} edges={tot} steps={steps} sha={dig}", flush=True)

"""Dev probe: TP class statistics of the C2 walks (groups and members per class)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
os.environ["ND_TP_TAIL"] = "0"
g = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
for name in ("node2vec", "ppr"):
    dr = run_device(make_app(name), g, n_samples=g.n_vertices, seed=7, paradigm="tp")
    st = dr.stats()
    a = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in st.timings])
    print(name, "steps", len(a), "groups small/medium/large total", a.sum(0).tolist(),
          "step0", a[0].tolist(), "step50", a[min(50, len(a) - 1)].tolist(), flush=True)
    dr.close()

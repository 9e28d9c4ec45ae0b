"""How much of a C2 TP walk runs in the staged hub tiers: the TP engine's
member counters (tp_staged = walker-steps sampled from a staged row in the
warp / thread-block tiers, tp_inplace = walker-steps stepped in place by the
sub-warp and grid tiers), per app, with the per-step class totals."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
out = {}
for name in ("node2vec", "ppr", "deepwalk"):
    dr = run_device(make_app(name), dg, n_samples=dg.n_vertices, seed=7, paradigm="tp")
    st = dr.stats()
    s, m, l = st.group_totals()
    c = dr.counters
    out[name] = {"tp_staged": c["tp_staged"], "tp_inplace": c["tp_inplace"],
                 "staged_share": c["tp_staged"] / max(1, c["tp_staged"] + c["tp_inplace"]),
                 "groups_small": s, "groups_medium": m, "groups_large": l,
                 "walker_steps": dr.total_sampled}
    dr.close()
print(json.dumps(out, indent=1))

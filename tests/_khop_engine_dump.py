"""Helper for test_fixed_layout_matches_step_loop: one k-hop configuration on
device, dumped to an .npz (run in a subprocess so ND_IND_FIXED can differ)."""
import sys

import numpy as np

sys.path.insert(0, sys.argv[1])
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.apps import UniformRoots  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

out_path, par, R, fan = sys.argv[2], sys.argv[3], int(sys.argv[4]), [int(x) for x in sys.argv[5].split(",")]
dg = DeviceGraph.rmat(11, 6, seed=9, undirected=False, weighted=False)  # directed: many dead ends
app = make_app("khop", fanouts=fan)
app.init_roots = UniformRoots(R)
dr = run_device(app, dg, n_samples=700, sample_lo=33, seed=12, paradigm=par)
o = dr.to_output()
off, ids = o.final_csr()
st = dr.stats()
cls = np.array([[t.groups_small, t.groups_medium, t.groups_large] for t in st.timings]).reshape(-1, 3)
np.savez(out_path, off=off, ids=ids, sc=o.step_counts, sv=o.step_vals, n_steps=o.n_steps, cls=cls,
         fetch=st.adjacency_fetches)

"""torchrun worker (not a test module) for tests/test_bench_multirank.py: multigpu.run_sharded on
two ranks (gloo collectives, both ranks on cuda:0); rank 0 compares the
gathered rows with a single-process run and writes the verdict to argv[1]."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.multigpu import run_sharded  # noqa: E402

dist.init_process_group("gloo")
torch.cuda.set_device(0)
g = DeviceGraph.rmat(12, 16, seed=3, weighted=True)
out = {}
for name in ("node2vec", "ppr", "khop"):
    app = make_app(name)
    off, ids = run_sharded(app, g, 5001, seed=9, paradigm="sp")
    if dist.get_rank() == 0:
        dr = run_device(app, g, n_samples=5001, seed=9, paradigm="sp")
        ref_off = dr.view(_lib.F_FINAL_OFF).cpu()
        ref_ids = dr.view(_lib.F_FINAL_IDS32).cpu()
        out[name] = bool(torch.equal(off.cpu(), ref_off) and torch.equal(ids.cpu(), ref_ids))
        dr.close()
if dist.get_rank() == 0:
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh)
dist.destroy_process_group()

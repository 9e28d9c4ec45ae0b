"""torchrun worker (not a test module) for tests/test_bench_multirank.py:
multigpu.ShardedJob (DeepWalk in 3 pieces per rank + k-hop, rows gathered to
rank 0 and copied to pinned host memory) on the ranks of the job (gloo
collectives, every rank on cuda:0); rank 0 puts the pieces back in sample-id
order, compares them with single-process runs and writes the verdict."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.multigpu import ShardedJob  # noqa: E402
from paper_2009_06693_b200.sharding import shard_for_rank, worker_ranges  # noqa: E402

dist.init_process_group("gloo")
torch.cuda.set_device(0)
ws, rank = dist.get_world_size(), dist.get_rank()
g = DeviceGraph.rmat(12, 16, seed=3, weighted=True)
N_DW, N_KH, CH = 5001, 777, 3
dw, kh = make_app("deepwalk"), make_app("khop", fanouts=[5, 3])
job = ShardedJob(g, [(dw, N_DW, 9, CH), (kh, N_KH, 9)], to_host=True)
for _ in range(2):  # pinned buffers are reused across runs
    res = job.run(order=[1, 0])
out = {}
if rank == 0:
    for (app, n, chunks), pieces in zip(((dw, N_DW, CH), (kh, N_KH, 1)), res):
        rows = {}
        for c, (off, ids) in enumerate(pieces):
            off, ids = off.numpy(), ids.numpy()
            r0 = 0
            for r in range(ws):
                lo, hi = shard_for_rank(n, ws, r)
                parts = worker_ranges(hi - lo, chunks) if hi > lo else []
                if c >= len(parts):
                    continue
                a, b = lo + parts[c][0], lo + parts[c][1]
                for sid in range(a, b):
                    rows[sid] = ids[off[r0]:off[r0 + 1]]
                    r0 += 1
            assert r0 == len(off) - 1
        dr = run_device(app, g, n_samples=n, seed=9, paradigm="sp")
        ref_off, ref_ids = dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)
        dr.close()
        out[app.name] = bool(len(rows) == n and all(
            np.array_equal(rows[i], ref_ids[ref_off[i]:ref_off[i + 1]]) for i in range(n)))
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh)
dist.destroy_process_group()

"""Dev probe: HostPipeline step time on C2 under ND_PIPE_NOCOPY / chunk settings."""
import statistics
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.streaming import HostPipeline  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
V = dg.n_vertices
apps = [make_app("node2vec", p=2.0, q=0.5), make_app("ppr", termination_probability=0.01)]
import ctypes as C  # noqa: E402
from paper_2009_06693_b200 import _lib  # noqa: E402
_d = torch.empty(V, dtype=torch.int64, device="cuda")
_lib.check(_lib.load().nd_uniform_roots(dg.handle, 1, C.c_uint64(7), 0, V, _lib.ptr(_d), _lib.stream_ptr()))
roots = _d.cpu().pin_memory()
def spec(x):  # "6" -> 6 chunks, "1:4:4:1" -> relative sizes
    return tuple(float(v) for v in x.split(":")) if ":" in x else int(x)


for cfg in sys.argv[1:] or ["6,3"]:
    c1, c2 = (spec(x) for x in cfg.split(","))
    pipe = HostPipeline(chunks=c1 if isinstance(c1, int) else len(c1))
    jobs = [(apps[0], V, 7, 0, roots, c1), (apps[1], V, 7, 0, roots, c2)]
    ms = []
    for it in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        pipe.run_jobs(dg, jobs)
        e.record()
        torch.cuda.synchronize()
        if it >= 2:
            ms.append(s.elapsed_time(e))
    print(cfg, os.environ.get("ND_PIPE_NOCOPY", "0"), round(statistics.median(ms), 2), flush=True)
    # pipelined: K runs back to back (wait=False), one wait at the end
    for K in (5,):
        for _ in range(2):  # both pinned buffer sets allocated
            pipe.run_jobs(dg, jobs, wait=False)
        pipe.wait()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(K):
            pipe.run_jobs(dg, jobs, wait=False)
        pipe.wait()
        e.record()
        torch.cuda.synchronize()
        print(cfg, "pipelined", K, round(s.elapsed_time(e) / K, 2), flush=True)

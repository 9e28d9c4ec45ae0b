"""Dev probe: the hub-bucket TP walk engine against the walker-major SP rows
and the sort-based TP engine's class statistics, plus timings.

  python tools/probe_tw.py [small|c1|c2 ...]
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import _lib, make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402
from paper_2009_06693_b200.synth import powerlaw_graph  # noqa: E402

APPS = [("deepwalk", {}), ("node2vec", {"p": 2.0, "q": 0.5}),
        ("ppr", {"termination_probability": 0.01})]


def run(app, g, n, par, env, reps):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ms = []
        for it in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dr = run_device(app, g, n_samples=n, seed=7, paradigm=par)
            e.record()
            torch.cuda.synchronize()
            ms.append(s.elapsed_time(e))
            if it < reps - 1:
                dr.close()
        out = {f: dr.host(f) for f in (_lib.F_FINAL_OFF, _lib.F_FINAL_IDS32, _lib.F_STATS,
                                       _lib.F_CHAIN_LEN)}
        out["steps"] = dr.n_steps
        dr.close()
        return statistics.median(ms), out
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    which = sys.argv[1:] or ["small", "c1"]
    graphs = []
    if "small" in which:
        graphs.append(("rmat14", DeviceGraph.rmat(14, 16, seed=1, weighted=True), 1 << 16))
        graphs.append(("rmat14u", DeviceGraph.rmat(14, 16, seed=2, weighted=False), 1 << 15))
    if "c1" in which:
        g = DeviceGraph.from_graph(powerlaw_graph(56944, attach=7, weighted=True, seed=0))
        graphs.append(("c1", g, g.n_vertices))
    if "c2" in which:
        g = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
        graphs.append(("c2", g, g.n_vertices))
    ok = True
    for gname, g, n in graphs:
        for aname, kw in APPS:
            app = make_app(aname, **kw)
            reps = 3
            t_sp, sp = run(app, g, n, "sp", {}, reps)
            t_hub0, hub0 = run(app, g, n, "tp", {"ND_TP_TAIL": "0"}, reps)
            t_hub, hub = run(app, g, n, "tp", {}, reps)
            t_srt, srt = run(app, g, n, "tp", {"ND_TP_TAIL": "0", "ND_TP_ENGINE": "sort"}, 1)
            rows_ok = all(np.array_equal(sp[f], hub0[f]) and np.array_equal(sp[f], hub[f])
                          for f in (_lib.F_FINAL_OFF, _lib.F_FINAL_IDS32, _lib.F_CHAIN_LEN))
            st_ok = np.array_equal(hub0[_lib.F_STATS], srt[_lib.F_STATS]) and \
                np.array_equal(hub[_lib.F_STATS], srt[_lib.F_STATS])
            ok &= rows_ok and st_ok
            print(f"{gname:8s} {aname:9s} n={n:8d} sp={t_sp:8.2f} tp-hub(all)={t_hub0:8.2f} "
                  f"tp-hub={t_hub:8.2f} tp-sort(all)={t_srt:8.2f} ms rows={'ok' if rows_ok else 'DIFF'} "
                  f"stats={'ok' if st_ok else 'DIFF'} steps={sp['steps']}/{hub0['steps']}/{srt['steps']}",
                  flush=True)
            if not st_ok:
                a, b = hub0[_lib.F_STATS].reshape(-1, 4), srt[_lib.F_STATS].reshape(-1, 4)
                print("  stats shapes", a.shape, b.shape)
                m = min(len(a), len(b))
                d = np.nonzero((a[:m] != b[:m]).any(1))[0][:5]
                for i in d:
                    print("  step", i, a[i], b[i])
    print("ALL OK" if ok else "MISMATCH")


if __name__ == "__main__":
    main()

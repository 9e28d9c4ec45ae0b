"""Dev probe: the C2 step's two apps (node2vec, PPR) in different launch
arrangements, event-timed medians of 7: one stream in either order, two
streams (the bench's run_device_concurrent), and two streams with one app's
stream at high priority."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_06693_b200 import make_app  # noqa: E402
from paper_2009_06693_b200.engine import run_device  # noqa: E402
from paper_2009_06693_b200.graph import DeviceGraph  # noqa: E402

dg = DeviceGraph.rmat(22, n_edges=68_993_773, seed=0, weighted=True)
N = dg.n_vertices
n2v, ppr = make_app("node2vec", p=2.0, q=0.5), make_app("ppr", termination_probability=0.01)
lo_pri, hi_pri = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two_streams(first, second, st_a, st_b):
    """each app on its own stream and host thread (a run synchronises its
    host thread between windows); the second thread starts 1 ms later"""
    import threading
    import time
    cur = torch.cuda.current_stream()
    st_a.wait_stream(cur)
    st_b.wait_stream(cur)
    out = [None, None]

    def go(k, app, st):
        with torch.cuda.stream(st):
            b = torch.cuda.Event(enable_timing=True)
            b.record(st)
            out[k] = run_device(app, dg, n_samples=N, seed=7, paradigm="sp", stream=st, sync=False)
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            TL.append((app.name, b, e))

    ta = threading.Thread(target=go, args=(0, first, st_a))
    tb = threading.Thread(target=go, args=(1, second, st_b))
    ta.start()
    time.sleep(0.001)
    tb.start()
    ta.join()
    tb.join()
    cur.wait_stream(st_a)
    cur.wait_stream(st_b)
    return out


def one_stream(first, second):
    a = run_device(first, dg, n_samples=N, seed=7, paradigm="sp", sync=False)
    b = run_device(second, dg, n_samples=N, seed=7, paradigm="sp", sync=False)
    return [a, b]


from paper_2009_06693_b200.engine import run_device_concurrent  # noqa: E402

variants = {
    "bench (run_device_concurrent n2v, ppr)": lambda: run_device_concurrent(
        [dict(app=n2v, n_samples=N, seed=7), dict(app=ppr, n_samples=N, seed=7)], dg),
    "serial n2v,ppr": lambda: one_stream(n2v, ppr),
    "serial ppr,n2v": lambda: one_stream(ppr, n2v),
    "2 streams n2v first": lambda: two_streams(n2v, ppr, s1, s2),
    "2 streams ppr first": lambda: two_streams(ppr, n2v, s1, s2),
    "ppr high priority, ppr first": lambda: two_streams(ppr, n2v, hi_pri, lo_pri),
    "n2v high priority, n2v first": lambda: two_streams(n2v, ppr, hi_pri, lo_pri),
    "ppr high priority, n2v first": lambda: two_streams(n2v, ppr, lo_pri, hi_pri),
}
TL = []
only = sys.argv[1:]
for name, fn in variants.items():
    if only and not any(o in name for o in only):
        continue
    for dr in fn():  # warm-up
        dr.close()
    torch.cuda.synchronize()
    ms = []
    for _ in range(int(os.environ.get("REPS", "7"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        runs = fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        if TL and os.environ.get("TIMELINE"):  # per app: [start, end] ms after the step's start
            print("  ", round(ms[-1], 2), [(a, round(e0.elapsed_time(b), 2), round(e0.elapsed_time(e), 2))
                                           for a, b, e in TL], flush=True)
        TL.clear()
        for dr in runs:
            dr.close()
    print(json.dumps({"variant": name, "ms_median": round(statistics.median(ms), 3),
                      "ms_min": round(min(ms), 3)}), flush=True)

#!/usr/bin/env python
"""Benchmark: sampled edges/s of the B200 NextDoor engine on the C2 workload.

Workload (BASELINE.json configs[1]): keyed RMAT scale 22
(4,194,304 vertices, 68,993,773 directed weighted edges, a,b,c = .57,.19,.19,
weights U[1,5), graph seed 0) built on device; one step = a node2vec walk
(p=2, q=0.5, length 100) plus a PPR walk (termination 0.01, step cap 10,000)
for every vertex (N = V walkers, sampling seed 7).  Inputs (1.4 GB CSR) are
larger than L2.  With --gpus N every rank builds the same keyed graph
(replicated, no broadcast) and runs its own block of sample ids: weak
scaling by default (each rank walks V walkers per app, global sample ids
[rank*V, (rank+1)*V): per-GPU work fixed, no collective on the data path,
the rows stay on the GPU that sampled them; --gather times the optional NCCL
gather of all rows to rank 0 separately).  --scaling strong splits the V
walkers with worker_ranges and gathers inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `value` = device throughput with inputs
resident (CUDA events, max over ranks); `e2e` = the same job through the
public API with host buffers (roots H2D, final rows D2H) in the timed
region; `roofline` = counted algorithmic bytes of the dominant kernel
(k_walk_persistent, SURVEY §8(d) sector model) / its event-timed duration;
`cpu_baseline` = the C oracle (restatement of the reference engine) on the
host's cores over a bounded sample of the same walks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

SCALE = 22
N_EDGES = 68_993_773
GRAPH_SEED = 0
SEED = 7
APPS = (("node2vec", {"p": 2.0, "q": 0.5}), ("ppr", {"termination_probability": 0.01}))
METRIC = "sampled edges/sec (and % of HBM roofline) at 1/2/4/8 B200 vs CPU ref"
CPU_SAMPLE = 1 << SCALE  # the full walker set: the C port runs it in ~10 s
DEV_SCALE = None  # --scale other than C2's (quick checks only)


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~5 ms from a background thread while the timed region runs (the timed
    region is ~0.1-0.2 s, shorter than nvidia-smi's start-up, so the CLI's
    `-lms` loop would see none of it).  The GPU is matched by UUID."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index=0, period_s=0.005):
        self.index = index
        self.period = period_s
        self.samples = []
        self.max_mhz = None
        self.error = None
        self._stop = threading.Event()
        self._thr = None
        self._nv = None
        self._h = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            self._nv = nv
            h = None
            try:
                uuid = str(torch.cuda.get_device_properties(index).uuid)
                for i in range(nv.nvmlDeviceGetCount()):
                    hh = nv.nvmlDeviceGetHandleByIndex(i)
                    u = nv.nvmlDeviceGetUUID(hh)
                    u = u.decode() if isinstance(u, bytes) else u
                    if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                        h = hh
                        break
            except Exception:
                h = None
            self._h = h if h is not None else nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
        except Exception as e:  # no NVML: the line says so
            self.error = f"nvml unavailable: {e}"

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((float(mhz), int(rs)))
            except Exception as e:
                self.error = str(e)
                return
            time.sleep(self.period)

    def __enter__(self):
        if self._h is not None:
            self._stop.clear()
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *a):
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=2)
            self._thr = None

    def summary(self):
        reasons = set()
        if self._nv is not None:
            for name, attr in self.REASONS:
                bit = getattr(self._nv, attr, 0)
                if any(r & bit for _, r in self.samples):
                    reasons.add(name)
        sm = [m for m, _ in self.samples]
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
               "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if self.error:
            out["error"] = self.error
        return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU: the oracle (C restatement of the reference engine) on host cores

def cpu_walks(hg, lo, n, threads):
    """Time node2vec + PPR for walkers [lo, lo+n) through the oracle's
    process-parallel-equivalent worker split (driver.py:175-186)."""
    from oracle import oracle as O
    og = O.OGraph(hg.n_vertices, hg.row_offsets, hg.col_indices, hg.weights,
                  hg.per_vertex_weight_prefix, hg.per_vertex_max_weight, None)
    roots = O.uniform_roots(hg.n_vertices, 1, SEED, lo, n)
    edges = 0
    res = {}
    t0 = time.perf_counter()
    for name, code, kp, steps in (("node2vec", 2, [2.0, 0.5, 0.0], 100), ("ppr", 1, [0.01], None)):
        r = O.run_chain(og, code, kp, roots, SEED, steps, paradigm="sp", n_threads=threads,
                        sample_lo=lo)
        vals = r["chain_vals"]
        edges += int((vals >= 0).sum())
        res[name] = r
    res["roots"] = np.asarray(roots).reshape(-1)
    return edges, time.perf_counter() - t0, res


def rows_equal_chain(off, ids, roots, r):
    """Device final rows (offsets, ids) == the oracle's chains, value for
    value: row i = roots[i] then chain i's non-NULL vertices in step order."""
    clen, cv = np.asarray(r["chain_len"]), np.asarray(r["chain_vals"])
    n = len(clen)
    starts = np.concatenate([[0], np.cumsum(clen)[:-1]]).astype(np.int64)
    ok = cv >= 0
    nn = np.add.reduceat(ok.astype(np.int64), starts) if len(cv) else np.zeros(n, np.int64)
    nn = np.where(clen > 0, nn, 0)
    if len(off) != n + 1 or not np.array_equal(np.diff(off), 1 + nn):
        return False
    exp = np.empty(int(off[-1]), dtype=np.int64)
    is_root = np.zeros(len(exp), dtype=bool)
    is_root[off[:-1]] = True
    exp[is_root] = roots
    exp[~is_root] = cv[ok]
    return bool(np.array_equal(np.asarray(ids, dtype=np.int64), exp))


def host_graph_for_oracle(dg):
    return dg.to_host()


# ---------------------------------------------------------------------------

def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def split_ranges(lo, n, parts):
    """worker_ranges (driver.py:175-186) of [lo, lo+n): contiguous, sizes
    differing by at most one, larger first."""
    parts = max(1, min(parts, n)) if n else 1
    base, extra = divmod(n, parts)
    out, a = [], lo
    for w in range(parts):
        b = a + base + (1 if w < extra else 0)
        out.append((a, b))
        a = b
    return out


# the reference itself (trawl, installed into baseline/_ref): forked worker
# processes share the graph copy-on-write (the process-parallel plan of
# BASELINE.md §3; the reference's own multi_worker_run, bench.py:123-153)
_REF = {}


def ref_trawl():
    """Import the installed reference (baseline/_ref) with its compiled
    kernels; (module, None) or (None, why)."""
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "trawl")):
        return None, "baseline/_ref/trawl is not installed"
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import trawl
    except Exception as e:  # noqa: BLE001
        return None, f"import trawl failed: {e}"
    if trawl.BACKEND_NAME != "compiled":
        return None, f"trawl backend is {trawl.BACKEND_NAME}, not compiled"
    return trawl, None


def _ref_task(rng):
    """One worker process: both apps over its sample-id range, each through
    the reference engine (sp_run / tp_run) with global sample ids."""
    trawl, g, engine = _REF["trawl"], _REF["graph"], _REF["engine"]
    from trawl.bench import _make_sample_range
    lo, hi = rng
    edges, eng_s = 0, 0.0
    for name, kw in APPS:
        app = trawl.make_app(name, **kw)
        samples = _make_sample_range(app, g, lo, hi, SEED)
        t0 = time.perf_counter()
        out = engine(app, g, samples, trawl.EngineConfig(seed=SEED, n_workers=1))
        eng_s += time.perf_counter() - t0
        edges += sum(s.total_sampled() for s in out.samples)
    return edges, eng_s


def trawl_walks(trawl, g, lo, n, procs, engine="sp"):
    """node2vec + PPR for sample ids [lo, lo+n) through the reference engine
    on `procs` forked processes.  Returns (edges, critical-path engine
    seconds = the slowest process, wall seconds)."""
    import multiprocessing as mp
    _REF.update(trawl=trawl, graph=g, engine=trawl.sp_run if engine == "sp" else trawl.tp_run)
    ranges = [r for r in split_ranges(lo, n, procs) if r[1] > r[0]]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(len(ranges)) as pool:
        res = pool.map(_ref_task, ranges, chunksize=1)
    wall = time.perf_counter() - t0
    return sum(r[0] for r in res), max(r[1] for r in res), wall


def trawl_graph(trawl, hg):
    """The reference's Graph over the same CSR arrays (prefix and max passed
    through: bit-identical to the reference's own, checked by the golden
    CSR tests)."""
    return trawl.Graph(hg.n_vertices, np.asarray(hg.row_offsets, dtype=np.int64),
                       np.asarray(hg.col_indices, dtype=np.int64),
                       np.asarray(hg.weights, dtype=np.float64),
                       np.arange(hg.n_vertices, dtype=np.int64),
                       per_vertex_max_weight=np.asarray(hg.per_vertex_max_weight),
                       per_vertex_weight_prefix=np.asarray(hg.per_vertex_weight_prefix))


REF_SAMPLE = 1 << 18  # walkers per app per reference-arm step (>= 2^17)


def run_reference(args):
    """--impl reference: the reference itself (trawl from baseline/_ref, its
    compiled kernels, sp_run) on all host cores in forked worker processes,
    over a bounded prefix of the same walks per step; the C oracle port
    timed beside it on the same sample.  The input graph is built on the
    host by the oracle's keyed RMAT generator and from_edges (the same CSR
    the GPU arm builds on device; no library of this repo is loaded)."""
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    cores = len(os.sched_getaffinity(0))
    from oracle import oracle as O
    scale = DEV_SCALE or SCALE
    t0 = time.perf_counter()
    src, dst, w = O.rmat_edges(scale, N_EDGES, seed=GRAPH_SEED, undirected=False, weighted=True)
    og = O.from_edges(src, dst, w, 1 << scale)
    del src, dst, w
    build_s = time.perf_counter() - t0
    sample = min(REF_SAMPLE, 1 << scale)
    trawl, why = ref_trawl()
    kind = "reference" if trawl is not None else "port"
    if trawl is not None:
        g = trawl_graph(trawl, og)
    times, walls, edges_tot = [], [], 0
    for i in range(args.warmup + args.steps):
        if trawl is not None:
            e, crit, wall = trawl_walks(trawl, g, 0, sample, cores, engine=args.ref_engine)
        else:
            e, crit, _ = cpu_walks(og, 0, sample, cores)
            wall = crit
        if i >= args.warmup:
            times.append(crit)
            walls.append(wall)
            edges_tot += e
    value = edges_tot / sum(times)
    # the oracle port on the same sample, for the record (and the check that
    # both CPU implementations sampled the same edges)
    pe, pdt, _ = cpu_walks(og, 0, sample, cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
        "config": config_dict(args.gpus, scaling=args.scaling),
        "cpu_baseline": {
            "value": value, "unit": "edges/s", "cores": cores, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": f"node2vec+PPR walks of sample ids [0, {sample}) per step "
                      f"({edges_tot // len(times)} edges)",
            "how": (f"trawl {args.ref_engine}_run (baseline/_ref, compiled kernels) in {cores} forked "
                    "processes over worker_ranges; time = slowest process's engine time"
                    if trawl is not None else f"C oracle port, {cores} threads ({why})"),
            "wall_ms_per_step": 1e3 * sum(walls) / len(walls),
            "port": {"value": pe / pdt, "cores": cores, "edges": pe,
                     "same_edges_as_reference": (pe == edges_tot // len(times))
                     if trawl is not None else None},
            "graph": f"keyed RMAT scale {scale} on the host (oracle rmat_edges + from_edges), "
                     f"{og.n_edges} edges, {build_s:.1f} s, outside the timed steps"},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(n_gpus, note=None, concurrent=True, scaling="weak"):
    weak = scaling == "weak"
    c = {"workload": "C2: RMAT scale 22 (4,194,304 V, 68,993,773 directed weighted E), "
                     "node2vec p=2 q=0.5 len 100 + PPR term 0.01, one walk per vertex"
                     + (" per GPU" if weak and n_gpus > 1 else ""),
         "graph": "keyed RMAT a=.57 b=.19 c=.19, weights U[1,5), seed 0, built on device",
         "walkers_per_step": 2 * (1 << (DEV_SCALE or SCALE)) * (n_gpus if weak else 1), "seed": SEED,
         "parallelism": (f"sample-sharded x{n_gpus}, graph replicated, "
                         + ("V walkers per app per GPU (ids rank*V..), no collective"
                            if weak else "V walkers split by worker_ranges, NCCL gather in the step")),
         "l2": "inputs (1.45 GB CSR) larger than L2", "paradigm": "sp (walker-major)",
         "apps": "node2vec and PPR concurrently on two streams" if concurrent else "node2vec then PPR"}
    if note:
        c["note"] = note
    if DEV_SCALE is not None:
        c["dev_scale"] = f"RMAT scale {DEV_SCALE}, {N_EDGES} edges: NOT the C2 workload"
    return c


# ---------------------------------------------------------------------------
# C5 (BASELINE.json configs[4]): DeepWalk + k-hop on the 1B-edge RMAT graph,
# the job split over the ranks (worker_ranges), rows gathered to rank 0

C5_SCALE, C5_EDGES, C5_WALKERS, C5_ROOTS = 26, 1 << 30, 1 << 23, 1 << 20


def c5_leg(args, ws, rank, barrier, rdev):
    """Strong-sharded C5 step through multigpu.ShardedJob: each rank builds the
    same keyed graph (replicated), runs its worker_ranges share of the 2^23
    DeepWalk walkers and the 2^20 k-hop (25, 10) roots concurrently, and sends
    each app's rows to rank 0 over NCCL as soon as the app finishes (k-hop
    first; its gather overlaps DeepWalk).  `value` includes the gather; `e2e`
    adds the roots' upload from pinned host memory on every rank and rank 0's
    copy of all gathered rows to pinned host memory."""
    import torch
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.multigpu import ShardedJob
    from paper_2009_06693_b200.sharding import shard_for_rank
    dev = DEV_SCALE is not None
    scale = DEV_SCALE if dev else C5_SCALE
    n_edges = (16 << scale) if dev else C5_EDGES
    walkers = (1 << (scale - 3)) if dev else C5_WALKERS
    roots = (1 << (scale - 6)) if dev else C5_ROOTS
    L = _lib.load()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg = DeviceGraph.rmat(scale, n_edges=n_edges, seed=GRAPH_SEED, weighted=True)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    dw, kh = make_app("deepwalk"), make_app("khop", fanouts=[25, 10])
    jobs = [(dw, walkers, SEED), (kh, roots, SEED)]
    order = [1, 0]  # k-hop finishes first: its rows travel while DeepWalk samples
    stream = torch.cuda.current_stream()

    step_times = []

    def timed_steps(job, k, w):
        last = None
        for _ in range(w):  # as in the timed steps, the previous step's rows stay alive
            last = job.run(order)
        barrier()
        times, edges = [], 0
        for _ in range(k):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            last = job.run(order)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            edges += job.last["edges"]
        ms = torch.tensor([sum(times)], dtype=torch.float64, device=rdev)
        ed = torch.tensor([edges], dtype=torch.int64, device=rdev)
        if ws > 1:
            torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
            torch.distributed.all_reduce(ed)
        step_times.append([round(t, 3) for t in times])  # this rank's, per step
        return ms.item(), int(ed.item()), last

    def checksum(rows):
        """Order-free checksum of rank 0's rows (the same at every N and chunking
        when the gathered rows equal the single-GPU run's): rows, values, the
        sum of the ids and of the squared row lengths."""
        out = {}
        for (app, n_total, _), pieces in zip(jobs, rows):
            c = {"rows": 0, "values": 0, "sum_ids": 0, "sum_len_sq": 0}
            for off, ids in pieces:
                ln = (off[1:] - off[:-1]).to(torch.int64)
                c["rows"] += int(ln.numel())
                c["values"] += int(ids.numel())
                c["sum_ids"] += int(ids.to(torch.int64).sum().item())
                c["sum_len_sq"] += int((ln * ln).sum().item())
            out[app.name] = c
        return out

    dev_job = ShardedJob(dg, jobs, to_host=False)
    dev_ms, dev_edges, rows = timed_steps(dev_job, args.steps, args.warmup)
    checks = checksum(rows) if rank == 0 else None
    del rows
    # e2e: DeepWalk's shard in pieces, so the rows of piece c cross PCIe while
    # piece c+1 samples
    host_jobs = [(dw, walkers, SEED, args.c5_chunks), (kh, roots, SEED)]
    host_job = ShardedJob(dg, host_jobs, to_host=True)
    e2e_ms, e2e_edges, hrows = timed_steps(host_job, args.steps, max(1, args.warmup // 2))
    e2e_checks = checksum(hrows) if rank == 0 else None
    h2d, d2h = host_job.last["h2d_bytes"], host_job.last["d2h_bytes"]
    del dev_job, host_job, hrows
    # each app's own kernel rate on this rank's shard (apps one after another,
    # event-timed launches; SURVEY 8(d) bytes counted on device)
    L.nd_set_profiling(1)
    kern = {}
    for app, n_total, _ in jobs:
        lo, hi = shard_for_rank(n_total, ws, rank)
        ms_k, b_k, e_k = 0.0, 0, 0
        for it in range(2):
            dr = run_device(app, dg, n_samples=hi - lo, sample_lo=lo, seed=SEED, paradigm="sp")
            if it:
                ms_k, b_k, e_k = dr.profile_ms[1], dr.counters["slot_bytes"], dr.total_sampled
            dr.close()
        kern[app.name] = (ms_k, b_k, e_k)
    L.nd_set_profiling(0)
    fp = dg.footprint()
    dg.close()
    torch.cuda.empty_cache()
    peak, peak_kind = peaks()
    roof = {}
    for name, (ms_k, b_k, e_k) in kern.items():
        gbs = b_k / (ms_k / 1e3) / 1e9 if ms_k > 0 else None
        roof[name] = {"kernel": "k_walk_persistent" if name == "deepwalk" else "k_fx_sample (fixed layout)",
                      "achieved": gbs, "peak": peak, "unit": "GB/s", "peak_kind": peak_kind,
                      "frac": gbs / peak if gbs else None, "kernel_ms": ms_k,
                      "algorithmic_bytes": b_k, "edges": e_k,
                      "edges_per_s": e_k / (ms_k / 1e3) if ms_k > 0 else None}
    return {
        "workload": (f"C5: RMAT scale {scale} ({dg.n_vertices:,} V, {dg.n_edges:,} directed weighted E), "
                     f"DeepWalk {walkers:,} walkers x 100 + k-hop (25,10) {roots:,} roots, "
                     f"split over {ws} GPU(s) by worker_ranges, rows gathered to rank 0 (NCCL)"
                     + ("" if not dev else " [dev scale: NOT C5]")),
        "value": dev_edges / (dev_ms / 1e3), "unit": "edges/s", "ms_per_step": dev_ms / args.steps,
        "step_ms_rank0": {"device": step_times[0], "e2e": step_times[1]},
        "scaling": "strong", "steps": args.steps, "warmup": args.warmup,
        "timing": "CUDA events around ShardedJob.run (sampling + NCCL gather of both apps' rows "
                  "to rank 0), max over ranks",
        "edges_per_step": dev_edges / args.steps,
        "e2e": {"value": e2e_edges / (e2e_ms / 1e3), "unit": "edges/s",
                "ms_per_step": e2e_ms / args.steps, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "result": "rank 0: every rank's final rows (int64 offsets + int32 ids) in pinned host memory",
                "chunks": {"deepwalk": args.c5_chunks, "khop": 1},
                "rows_match_device": e2e_checks == checks if rank == 0 else None,
                "timing": "roots H2D on every rank + sampling + NCCL gather + rank-0 D2H, per step"},
        "rows_on_rank0": checks,
        "per_rank_kernels": roof,
        "graph": {"build_s": build_s, **fp},
        "note": "strong scaling: the same 2^23 + 2^20 samples at every N; the checksums of rank 0's "
                "rows are identical at every N when the gathered rows equal the 1-GPU run",
    }


def _timed_runs(app, dg, lo, n, par, reps=5, warm=2):
    """Median event time of whole runs (sampling, inversion, compaction) of
    this rank's block, and the last run's sampled / recorded counts."""
    import torch
    from paper_2009_06693_b200.engine import run_device
    stream = torch.cuda.current_stream()
    for _ in range(warm):
        run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm=par).close()
    ms, sampled, recorded = [], 0, 0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dr = run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm=par, sync=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        sampled, recorded = dr.total_sampled, dr.total_recorded
        dr.close()
    return statistics.median(ms), sampled, recorded


def _rank_max_sum(ms, cnt, ws, rdev):
    import torch
    a = torch.tensor([ms], dtype=torch.float64, device=rdev)
    b = torch.tensor([cnt], dtype=torch.int64, device=rdev)
    if ws > 1:
        torch.distributed.all_reduce(a, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(b)
    return a.item(), int(b.item())


def c1_c4_legs(args, ws, rank, barrier, rdev):
    """C1 (BASELINE.json configs[0]: DeepWalk x 56,944 on the reference's own
    powerlaw(56944, attach 7) graph, L2-resident) and C4 (configs[3]:
    FastGCN / LADIES (deg^2) / MVS over 4,096 samples and ClusterGCN over 8
    on the Orkut-shaped RMAT-22 graph, 117.2M directed unit edges), each
    rank its worker_ranges block; median event times of whole runs.  Parity
    of these configurations is in tests/test_gpu_configs.py."""
    import torch
    from paper_2009_06693_b200 import make_app
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.sharding import shard_for_rank
    from paper_2009_06693_b200.synth import powerlaw_graph
    out = {}
    g = powerlaw_graph(56944, attach=7, weighted=True, seed=0)
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.weights)
    lo, hi = shard_for_rank(g.n_vertices, ws, rank)
    c1 = {"workload": "C1: DeepWalk len 100, one walk per vertex, powerlaw(56944, attach 7, "
                      "weighted, seed 0): 797,132 edges, L2-resident (HBM roofline not binding)"}
    for par in ("sp", "tp"):
        ms, e, _ = _timed_runs(make_app("deepwalk"), dg, lo, hi - lo, par)
        ms, e = _rank_max_sum(ms, e, ws, rdev)
        c1[par] = {"ms": ms, "edges": e, "value": e / (ms / 1e3), "unit": "edges/s"}
    c1["graph_footprint"] = dg.footprint()
    dg.close()
    out["c1"] = c1
    if DEV_SCALE is None:
        dg = DeviceGraph.rmat(22, n_edges=58_600_000, seed=GRAPH_SEED, undirected=True, weighted=False)
    else:
        dg = DeviceGraph.rmat(DEV_SCALE, n_edges=int(58_600_000 / (1 << 22) * (1 << DEV_SCALE)),
                              seed=GRAPH_SEED, undirected=True, weighted=False)
    c4 = {"workload": f"C4: collective apps on RMAT scale {DEV_SCALE or 22} "
                      f"({dg.n_vertices:,} V, {dg.n_edges:,} directed unit E), tp_run's engine",
          "unit": "sampled + recorded edges/s"}
    for name, kw, N in (("fastgcn", {}, 4096), ("ladies", {"distribution": "degree_sq"}, 4096),
                        ("mvs", {}, 4096), ("clustergcn", {}, 8)):
        lo, hi = shard_for_rank(N, ws, rank)
        if hi > lo:
            ms, smp, rec = _timed_runs(make_app(name, **kw), dg, lo, hi - lo, "tp", reps=3, warm=1)
        else:
            ms, smp, rec = 0.0, 0, 0
        ms, smp = _rank_max_sum(ms, smp, ws, rdev)
        _, rec = _rank_max_sum(0.0, rec, ws, rdev)
        c4[name] = {"N": N, "ms": ms, "sampled": smp, "recorded": rec,
                    "value": (smp + rec) / (ms / 1e3) if ms > 0 else None}
    c4["graph_footprint"] = dg.footprint()
    dg.close()
    torch.cuda.empty_cache()
    out["c4"] = c4
    return out


def c3_leg(args, ws, rank, barrier, rdev):
    """C3 (BASELINE.json configs[2]): GraphSAGE k-hop (25, 10) on the
    Reddit-shaped RMAT-18 graph (57.3M undirected edges, 114.6M directed, unit
    weights), 228 batches of 1024 roots as one launch, this rank's
    worker_ranges share; SP (fixed layout) and TP (hub-bucket inversion)
    event-timed, the sampling kernels' §8(d) bytes against the HBM peak."""
    import torch
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import profiling, run_device
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.sharding import shard_for_rank
    dev = DEV_SCALE is not None
    scale = min(DEV_SCALE, 18) if dev else 18
    dg = DeviceGraph.rmat(scale, n_edges=int(57_300_000 / (1 << 18) * (1 << scale)), seed=GRAPH_SEED,
                          undirected=True, weighted=False)
    app = make_app("khop", fanouts=[25, 10])
    N = 1024 * 228
    lo, hi = shard_for_rank(N, ws, rank)
    stream = torch.cuda.current_stream()
    peak, peak_kind = peaks()
    out = {"workload": f"C3: k-hop (25,10), {N:,} roots (228 x 1024) on RMAT scale {scale} "
                       f"({dg.n_vertices:,} V, {dg.n_edges:,} directed unit E), split over {ws} GPU(s)"
                       + (" [dev scale: NOT C3]" if dev else "")}
    for par in ("sp", "tp"):
        for _ in range(3):
            run_device(app, dg, n_samples=hi - lo, sample_lo=lo, seed=SEED, paradigm=par).close()
        ms_l, edges = [], 0
        for _ in range(5):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dr = run_device(app, dg, n_samples=hi - lo, sample_lo=lo, seed=SEED, paradigm=par,
                            sync=False)
            e1.record(stream)
            torch.cuda.synchronize()
            ms_l.append(e0.elapsed_time(e1))
            edges = dr.total_sampled
            dr.close()
        with profiling():
            dr = run_device(app, dg, n_samples=hi - lo, sample_lo=lo, seed=SEED, paradigm=par)
        k_ms, k_bytes, steps = dr.profile_ms[1], dr.counters["slot_bytes"], dr.step_ms
        dr.close()
        ms = torch.tensor([statistics.median(ms_l)], dtype=torch.float64, device=rdev)
        ed = torch.tensor([edges], dtype=torch.int64, device=rdev)
        if ws > 1:
            torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
            torch.distributed.all_reduce(ed)
        gbs = k_bytes / (k_ms / 1e3) / 1e9 if k_ms > 0 else None
        # measured DRAM bytes of the same sampling kernels per run (the
        # newest committed ncu capture of this workload, tools/ncu_round.sh)
        dram = None
        try:
            import glob
            prof = sorted(glob.glob(os.path.join(REPO, "profiles", "r*_ncu_summary.json")))[-1]
            kh = json.load(open(prof))["workloads"]["khop"]
            names = ["k_fx_sample"] if par == "sp" else ["k_fx_small", "k_fx_hub_warp",
                                                        "k_fx_hub_cta<4>"]
            # the capture holds one SP run and one TP run: both steps' launches of each
            b_run = sum(kh[k]["dram_bytes"] for k in names if k in kh)
            dram = {"bytes_per_run": b_run, "gbs": b_run / (k_ms / 1e3) / 1e9 if k_ms > 0 else None,
                    "frac": b_run / (k_ms / 1e3) / 1e9 / peak if k_ms > 0 else None,
                    "source": os.path.relpath(prof, REPO)}
        except Exception:
            dram = None
        out[par] = {"ms": ms.item(), "edges": int(ed.item()),
                    "value": int(ed.item()) / (ms.item() / 1e3), "unit": "edges/s",
                    "timing": "median of 5 event-timed whole runs (sampling, inversion, compaction)",
                    "roofline": {"achieved": gbs, "peak": peak, "unit": "GB/s", "peak_kind": peak_kind,
                                 "frac": gbs / peak if gbs else None,
                                 "kernel_ms": k_ms, "algorithmic_bytes": k_bytes,
                                 "step_build_sample_ms": steps,
                                 "kernels": "k_fx_sample" if par == "sp" else
                                            "k_fx_small + k_fx_hub_warp + k_fx_hub_cta",
                                 "dram": dram}}
    out["tp_vs_sp"] = out["tp"]["ms"] / out["sp"]["ms"]
    out["graph_footprint"] = dg.footprint()
    # single 1,024-root batches (report C3's batch latency):
    # run_device per batch vs the CUDA-graph plan (minibatch.KhopBatchSampler)
    # replayed over 228 batches back to back, keyed roots of each batch's ids
    import ctypes as C
    from paper_2009_06693_b200.minibatch import KhopBatchSampler
    nb, bs = 228, 1024
    L = _lib.load()
    allroots = torch.empty(nb * bs, dtype=torch.int64, device="cuda")
    _lib.check(L.nd_uniform_roots(dg.handle, 1, C.c_uint64(SEED), 0, nb * bs, _lib.ptr(allroots),
                                  _lib.stream_ptr()), "nd_uniform_roots")
    one = []
    for b in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dr = run_device(app, dg, n_samples=bs, sample_lo=b * bs, seed=SEED, paradigm="sp", sync=False)
        e1.record(stream)
        torch.cuda.synchronize()
        if b >= 5:
            one.append(e0.elapsed_time(e1))
        dr.close()
    sampler = KhopBatchSampler(dg, [25, 10], bs)
    for b in range(5):
        sampler.sample(allroots[b * bs:(b + 1) * bs], sample_lo=b * bs, seed=SEED)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    edges = 0
    e0.record(stream)
    for b in range(nb):
        off, _, _ = sampler.sample(allroots[b * bs:(b + 1) * bs], sample_lo=b * bs, seed=SEED)
    e1.record(stream)
    torch.cuda.synchronize()
    plan_ms = e0.elapsed_time(e1) / nb
    # the last batch's rows equal a plain run of it
    dr = run_device(app, dg, n_samples=bs, sample_lo=(nb - 1) * bs, seed=SEED, paradigm="sp")
    same = bool(torch.equal(off, dr.view(_lib.F_FINAL_OFF))
                and torch.equal(sampler.final_ids[:int(off[-1])], dr.view(_lib.F_FINAL_IDS32)))
    edges = dr.total_sampled
    dr.close()
    sampler.close()
    out["single_batch"] = {"roots": bs, "edges": edges,
                           "run_device_ms": statistics.median(one),
                           "plan_ms": plan_ms, "plan_edges_per_s": edges / (plan_ms / 1e3),
                           "plan_rows_equal_run": same,
                           "how": "run_device: median of 20 event-timed single-batch runs; plan: "
                                  f"{nb} batches replayed back to back (one CUDA graph launch each), "
                                  "event time / batches"}
    dg.close()
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--paradigm", default="sp", choices=["sp", "tp"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tp", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (1B-edge, strong-sharded) leg")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 (k-hop) leg")
    ap.add_argument("--no-c14", action="store_true", help="skip the C1 (DeepWalk) and C4 (collective) legs")
    ap.add_argument("--c5-chunks", type=int, default=8,
                    help="C5 e2e: DeepWalk pieces per rank (piece c's rows cross PCIe while c+1 samples)")
    ap.add_argument("--ref-engine", default="sp", choices=["sp", "tp"],
                    help="the reference engine timed by --impl reference (sp_run: its faster CPU path)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--gather", action="store_true",
                    help="also time an NCCL gather of every rank's rows to rank 0 (reported separately)")
    ap.add_argument("--serial-apps", action="store_true",
                    help="run node2vec then PPR instead of concurrently on two streams")
    ap.add_argument("--e2e-chunks", type=int, default=2,
                    help="node2vec sample-id chunks of the host pipeline (D2H of chunk c overlaps chunk c+1)")
    ap.add_argument("--e2e-ppr-chunks", type=int, default=1)
    ap.add_argument("--scale", type=int, default=SCALE,
                    help="RMAT scale (22 = C2; smaller only for quick multi-rank checks)")
    args = ap.parse_args()
    if args.scale != SCALE:  # development scale: same mean degree, flagged in config
        global N_EDGES, CPU_SAMPLE, DEV_SCALE
        DEV_SCALE = args.scale
        N_EDGES = int(N_EDGES / (1 << SCALE) * (1 << args.scale))
        CPU_SAMPLE = 1 << args.scale
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    backend = os.environ.get("ND_DIST_BACKEND", "nccl")  # gloo: multi-rank check on one GPU
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2009_06693_b200 import _lib, make_app
    from paper_2009_06693_b200.engine import job_streams, run_device, submit_device_concurrent
    from paper_2009_06693_b200.graph import DeviceGraph
    from paper_2009_06693_b200.sharding import worker_ranges

    L = _lib.load()
    dg = DeviceGraph.rmat(DEV_SCALE or SCALE, n_edges=N_EDGES, seed=GRAPH_SEED, weighted=True)
    V = dg.n_vertices
    if args.scaling == "weak":  # per-GPU work fixed: this rank's own V walkers per app
        lo, n = rank * V, V
    else:
        lo, hi = worker_ranges(V, ws)[rank] if rank < min(ws, V) else (V, V)
        n = hi - lo
    gather_in_step = ws > 1 and args.scaling == "strong"
    apps = [make_app(a, **kw) for a, kw in APPS]
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    def gather_rows(off, ids):
        """Final NCCL gather of every rank's compacted rows to rank 0."""
        if ws == 1:
            return 0
        from paper_2009_06693_b200.multigpu import gather_rows as g
        g(off, ids)
        return 0

    # ---- device throughput: inputs resident, CUDA events, max over ranks --------
    L.nd_set_profiling(1)
    sample_ms, slot_bytes, edges_dev, launches, rand_sect = [], 0, 0, 0, 0
    times = []
    clocks = ClockSampler(local)
    for it in range(args.warmup + args.steps):
        timed = it >= args.warmup
        if timed and it == args.warmup:
            clocks.__enter__()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        step_edges, step_bytes, step_sample, step_sect = 0, 0, 0.0, 0
        runs = []
        if args.serial_apps:
            for app in apps:
                runs.append(run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED,
                                       paradigm=args.paradigm, sync=False))
                if gather_in_step:
                    gather_rows(runs[-1].view(_lib.F_FINAL_OFF), runs[-1].narrow_ids())
        else:  # node2vec and PPR concurrently (PPR's long-walk tail overlaps node2vec)
            futs = submit_device_concurrent([dict(app=app, n_samples=n, sample_lo=lo, seed=SEED)
                                             for app in apps], dg, paradigm=args.paradigm)
            for fut, st in zip(futs, job_streams(len(apps))):
                runs.append(fut.result())
                stream.wait_stream(st)
                if gather_in_step:  # this app's rows go to rank 0 while the other app samples
                    gather_rows(runs[-1].view(_lib.F_FINAL_OFF), runs[-1].narrow_ids())
        for dr in runs:
            step_edges += dr.total_sampled
            step_bytes += dr.counters["slot_bytes"]
            step_sect += dr.counters.get("rand_sectors", 0)
            step_sample += dr.profile_ms[1]
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        for dr in runs:
            dr.close()
        if os.environ.get("ND_BENCH_VERBOSE"):
            print(json.dumps({"it": it, "ms": ms, "per_app_prof": [dr.profile_ms for dr in runs]}),
                  file=sys.stderr, flush=True)
        if timed:
            times.append(ms)
            edges_dev += step_edges
            slot_bytes += step_bytes
            rand_sect += step_sect
            sample_ms.append(step_sample)
            launches += sum(int(dr.counters.get("launches", 0)) for dr in runs)
    clocks.__exit__()
    tot_ms = sum(times)
    rdev = "cuda" if backend == "nccl" else "cpu"
    if ws > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = t.item()
        e = torch.tensor([edges_dev], dtype=torch.int64, device=rdev)
        dist.all_reduce(e)
        edges_all = int(e.item())
    else:
        edges_all = edges_dev
    value = edges_all / (tot_ms / 1e3)

    # ---- optional: NCCL gather of every rank's rows to rank 0 (not in `value`) -------
    gather_info = None
    if args.gather and ws > 1 and args.scaling == "weak":
        runs = [run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm=args.paradigm)
                for app in apps]
        nbytes = 0
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for dr in runs:
            off, ids = dr.view(_lib.F_FINAL_OFF), dr.narrow_ids()
            nbytes += off.numel() * 8 + ids.numel() * 4
            gather_rows(off, ids)
        g1.record(stream)
        torch.cuda.synchronize()
        gms = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        for dr in runs:
            dr.close()
        gather_info = {"ms": gms.item(), "bytes_per_rank": nbytes, "backend": backend,
                       "note": "int32 rows of both apps gathered to rank 0 after the timed steps"}

    # ---- the transit-parallel paradigm on the same job (reported alongside) ----------
    # tp_run's engine (nd_walk_hub.cuh): per step, member counts fused into the
    # previous step's emission, hub tiers, staged rows; the same two apps
    # concurrently on two streams as the SP step, then each app alone
    tp_info = None
    if args.paradigm == "sp" and not args.no_tp:
        from paper_2009_06693_b200.engine import run_device_concurrent
        tp_ms, tp_app = [], {a.name: [] for a in apps}
        tp_rows_equal = None
        for it in range(3):
            barrier()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            runs = run_device_concurrent([dict(app=app, n_samples=n, sample_lo=lo, seed=SEED)
                                          for app in apps], dg, paradigm="tp")
            ev1.record(stream)
            torch.cuda.synchronize()
            if it:
                tp_ms.append(ev0.elapsed_time(ev1))
            else:  # the TP rows equal the SP rows (checked once, on device)
                sp_runs = run_device_concurrent([dict(app=app, n_samples=n, sample_lo=lo, seed=SEED)
                                                 for app in apps], dg, paradigm="sp")
                tp_rows_equal = all(
                    torch.equal(a.view(_lib.F_FINAL_OFF), b.view(_lib.F_FINAL_OFF))
                    and torch.equal(a.narrow_ids(), b.narrow_ids())
                    for a, b in zip(runs, sp_runs))
                for dr in sp_runs:
                    dr.close()
            for dr in runs:
                dr.close()
        for it in range(2):
            for app in apps:
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm="tp").close()
                ev1.record(stream)
                torch.cuda.synchronize()
                tp_app[app.name].append(ev0.elapsed_time(ev1))
        tp_step = sum(tp_ms) / len(tp_ms)
        tp_info = {"ms_per_step": tp_step,
                   "value": (edges_dev / len(times)) / (tp_step / 1e3),
                   "vs_sp": tp_step / (sum(times) / len(times)),
                   "ms_per_app_alone": {k: min(v) for k, v in tp_app.items()},
                   "rows_equal_sp": tp_rows_equal,
                   "note": "tp_run's engine: per step, member counts fused into the previous step's "
                           "emission (exact class statistics), prep of the hub tiers, sub-warp + "
                           "grid tiers stepped in place, warp / thread-block tiers from rows staged "
                           "by bulk copy; walker-major tail with exact class statistics below "
                           "131,072 alive walkers; both apps concurrently as in the SP step"}

    # ---- e2e through the public API with host buffers ------------------------------
    # HostPipeline (paper_2009_06693_b200/streaming.py): roots uploaded from
    # pinned host memory per chunk, final rows (int64 offsets + int32 ids)
    # copied back into pinned host buffers while the next chunk samples.
    L.nd_set_profiling(0)
    from paper_2009_06693_b200.streaming import HostPipeline
    # the step's input: the keyed default roots (apps.py:83-103) as a host
    # array, produced once by the library (nd_uniform_roots) outside the timed steps
    import ctypes as C
    droots = torch.empty(n, dtype=torch.int64, device="cuda")
    _lib.check(L.nd_uniform_roots(dg.handle, 1, C.c_uint64(SEED), lo, n, _lib.ptr(droots),
                                  _lib.stream_ptr()), "nd_uniform_roots")
    roots_host = droots.cpu().pin_memory()
    del droots
    e2e_edges, h2d, d2h = 0, 0, 0
    e2e_ok = True
    pipe = HostPipeline(chunks=args.e2e_chunks)
    # fixed-length node2vec splits into chunks freely; PPR's chunks each repeat
    # its latency-bound tail window, so it takes fewer and overlaps node2vec
    chunk_of = {"node2vec": args.e2e_chunks, "ppr": args.e2e_ppr_chunks}
    jobs = [(app, n, SEED, lo, roots_host, chunk_of.get(app.name, args.e2e_chunks)) for app in apps]
    for it in range(max(1, args.warmup // 2)):  # warm-up, waited; the first checks the rows
        res = pipe.run_jobs(dg, jobs)
        if it == 0:  # host rows == device rows of a plain run (checksums, outside the timed steps)
            for app, chunks in zip(apps, res):
                dr = run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm=args.paradigm)
                ref_ids = dr.view(_lib.F_FINAL_IDS)
                e2e_ok &= bool(sum(int(c.ids.sum()) for c in chunks) == int(ref_ids.sum().item()))
                e2e_ok &= bool(sum(c.ids.numel() for c in chunks) == ref_ids.numel())
                dr.close()
    for _ in range(2):  # both pinned buffer sets of the back-to-back mode allocated
        pipe.run_jobs(dg, jobs, wait=False)
    pipe.wait()
    # K steps back to back (step k+1 samples while step k's last rows cross
    # PCIe), bracketed by a barrier + synchronize; every step uploads its roots
    # and copies all its rows into pinned host memory
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for it in range(args.steps):
        res = pipe.run_jobs(dg, jobs, wait=False)
        e2e_edges += sum(c.total_sampled for chunks in res for c in chunks)
        h2d = pipe.last_h2d_bytes  # the roots, uploaded once for both apps
        d2h = sum(c.offsets.numel() * c.offsets.element_size() + c.ids.numel() * c.ids.element_size()
                  for chunks in res for c in chunks)
    pipe.wait()
    ev1.record(stream)
    torch.cuda.synchronize()
    e2e_times = [ev0.elapsed_time(ev1)]
    e2e_ms = sum(e2e_times)
    if ws > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
        e = torch.tensor([e2e_edges], dtype=torch.int64, device=rdev)
        dist.all_reduce(e)
        e2e_edges = int(e.item())
    e2e_value = e2e_edges / (e2e_ms / 1e3)

    # ---- roofline of the dominant kernel ----------------------------------------------
    # The timed steps run the two apps concurrently, so a launch's event time
    # there includes the other app's share of the GPU.  The kernel's own rate
    # comes from a separate pass with the apps one after another (same
    # kernels, same inputs, event-timed launches on their stream).
    peak, peak_kind = peaks()
    L.nd_set_profiling(1)
    rf_ms, rf_bytes, rf_sect = 0.0, 0, 0
    for it in range(3):
        for app in apps:
            dr = run_device(app, dg, n_samples=n, sample_lo=lo, seed=SEED, paradigm=args.paradigm)
            if it:
                rf_ms += dr.profile_ms[1]
                rf_bytes += dr.counters["slot_bytes"]
                rf_sect += dr.counters.get("rand_sectors", 0)
            dr.close()
    L.nd_set_profiling(0)
    samp_s = rf_ms / 1e3
    achieved = (rf_bytes / samp_s / 1e9) if samp_s > 0 else None
    # DRAM bytes of the same kernel launches from the newest committed
    # `ncu --set full` capture of this code (tools/ncu_walk.sh writes it each
    # round; ncu cannot run inside the timed bench)
    traffic, traffic_src = None, None
    import glob
    for prof_json in sorted(glob.glob(os.path.join(REPO, "profiles", "r*_ncu_summary.json")),
                            reverse=True):
        try:
            with open(prof_json) as fh:
                traffic = json.load(fh).get("traffic_bytes_per_step")
            traffic_src = os.path.relpath(prof_json, REPO)
            break
        except Exception:
            traffic = None
    # the random-gather ceiling of this GPU (nd_gather_ceiling: dependent random
    # 32-byte sector reads over a buffer the size of the graph's records), the
    # roofline a gather-bound walk actually faces beside the copy peak
    import ctypes as C
    ceil = C.c_double(0.0)
    ceil_bytes = int(min(dg.resident_bytes(), 8 << 30))
    gather = None
    if L.nd_gather_ceiling(ceil_bytes, 4, 64, C.byref(ceil), _lib.stream_ptr()) == 0 and samp_s > 0:
        rate = rf_sect / samp_s
        gather = {"sectors_per_s": rate, "ceiling_sectors_per_s": ceil.value,
                  "frac": rate / ceil.value if ceil.value else None,
                  "ceiling_how": f"dependent random 32 B reads, 1 chain/thread, 4x256 threads/SM, "
                                 f"{ceil_bytes / 2**30:.1f} GiB buffer (nd_gather_ceiling)",
                  "sectors": "random 32 B sector reads counted on device by the walk kernels"}

    # ---- CPU baseline (rank 0, N=1 only) ------------------------------------------------
    cpu = None
    parity = None
    parity_values = 0
    if rank == 0 and ws == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        hg = host_graph_for_oracle(dg)
        ce, cdt, cres = cpu_walks(hg, 0, CPU_SAMPLE, cores)
        port = {"value": ce / cdt, "unit": "edges/s", "cores": cores, "kind": "port",
                "sample": f"node2vec+PPR walks for sample ids [0, {CPU_SAMPLE}) "
                          f"({ce} edges, {cdt:.1f} s)", "threads": cores}
        cpu = dict(port)
        # the reference itself (trawl from baseline/_ref) on the same cores,
        # forked worker processes over a bounded prefix
        trawl, why = ref_trawl()
        if trawl is not None:
            re_, crit, wall = trawl_walks(trawl, trawl_graph(trawl, hg), 0,
                                          min(REF_SAMPLE, CPU_SAMPLE), cores)
            cpu = {"value": re_ / crit, "unit": "edges/s", "cores": cores, "kind": "reference",
                   "sample": f"node2vec+PPR walks for sample ids [0, {min(REF_SAMPLE, CPU_SAMPLE)}) "
                             f"({re_} edges)",
                   "how": f"trawl sp_run (baseline/_ref, compiled kernels) in {cores} forked "
                          "processes over worker_ranges; time = slowest process's engine time",
                   "wall_s": wall, "port": port}
        else:
            cpu["reference_unavailable"] = why
        cpu["cpu_model"] = cpu_model()
        # parity of every sampled row on the CPU sample: offsets and every
        # vertex id (root, then the walk's non-NULL steps, chain.py:166-179)
        parity = True
        for (name, kw), app in zip(APPS, apps):
            dr = run_device(app, dg, n_samples=CPU_SAMPLE, seed=SEED, paradigm=args.paradigm)
            off, ids = dr.host(_lib.F_FINAL_OFF), dr.host(_lib.F_FINAL_IDS)
            dr.close()
            parity &= bool(rows_equal_chain(off, ids, cres["roots"], cres[name]))
        parity_values = int(sum(len(cres[k]["chain_vals"]) for k in ("node2vec", "ppr")))

    c2_footprint = dg.footprint()
    dg.close()
    torch.cuda.empty_cache()
    # every leg starts from a trimmed allocation pool (the C2 legs leave it
    # shaped by multi-GB windows; the k-hop TP steps measured 5% slower on it)
    L.nd_pool_trim(0)
    c3 = None if args.no_c3 else c3_leg(args, ws, rank, barrier, rdev)
    L.nd_pool_trim(0)
    c14 = {} if args.no_c14 else c1_c4_legs(args, ws, rank, barrier, rdev)
    L.nd_pool_trim(0)
    c5 = None
    if not args.no_c5:
        c5 = c5_leg(args, ws, rank, barrier, rdev)

    if rank == 0:
        ms_per_step = tot_ms / len(times)
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "int64+f64", "data": "synthetic",
            "config": config_dict(ws, concurrent=not args.serial_apps, scaling=args.scaling),
            "e2e": {"value": e2e_value, "unit": "edges/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "host_rows_match_device": e2e_ok,
                    "result": "final rows: int64 offsets + int32 vertex ids, pinned host",
                    "chunks": {"node2vec": args.e2e_chunks, "ppr": args.e2e_ppr_chunks},
                    "ms_per_step": e2e_ms / args.steps,
                    "timing": "K steps back to back through HostPipeline.run_jobs(wait=False) "
                              "(step k+1 samples while step k's last rows cross PCIe), "
                              "barrier + synchronize around all K"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         # traffic is per step; samp_s covers the 2 timed passes
                         "dram_gbs": (traffic / (samp_s / 2) / 1e9) if (traffic and samp_s > 0) else None,
                         "dram_frac": (traffic / (samp_s / 2) / 1e9 / peak) if (traffic and samp_s > 0)
                         else None,
                         "kernel": "k_walk_persistent" if args.paradigm == "sp" else "TP class kernels",
                         "peak_kind": peak_kind,
                         "bytes_model": "SURVEY 8(d) sector model, counted on device",
                         "algorithmic_bytes_per_step": slot_bytes / len(times),
                         "kernel_ms_per_step": rf_ms / 2,
                         "kernel_timing": "apps one after another (2 passes), event-timed launches",
                         # the timed step runs both apps' kernels side by side (each on
                         # half of every SM's CTA slots): their combined algorithmic
                         # bytes over the whole step time (a lower bound, the step also
                         # holds the roots, the compaction and the host syncs)
                         "step_achieved": (slot_bytes / len(times)) / (sum(times) / len(times) / 1e3) / 1e9,
                         "step_frac": (slot_bytes / len(times)) / (sum(times) / len(times) / 1e3) / 1e9
                         / peak,
                         "gather": gather},
            "cpu_baseline": cpu, "parity_cpu_sample": parity,
            "parity": {"ok": parity, "values_compared": parity_values if parity is not None else 0,
                       "how": "every final-row offset and vertex id of the CPU sample's walkers "
                              "(both apps) equals the C oracle's"} if parity is not None else None,
            "paradigm_tp": tp_info,
            "clocks": clocks.summary(), "gpu_launches": launches, "gather": gather_info,
            "edges_per_step": edges_all / len(times),
            "graph_footprint": c2_footprint,
            "c1": c14.get("c1"),
            "c3": c3,
            "c4": c14.get("c4"),
            "c5": c5,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

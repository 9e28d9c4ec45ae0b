"""Host-streaming runs: sample rows delivered to pinned host memory while the
device samples the next chunk.

The reference hands a finished ``SampleSetOutput`` back to the caller
(``tp_run``/``sp_run``, transit_parallel.py:249-257; the CLI then renders it,
cli.py:95-137).  On B200 the device samples several times faster than PCIe
can carry the rows back, so a run to host memory is split into contiguous
sample-id chunks (the keyed RNG makes any split produce identical rows,
driver.py:175-186): while chunk c+1 runs on the compute stream, chunk c's
final rows (int64 offsets + int32 vertex ids) are copied device->host on a
copy stream into caller-owned pinned buffers.  Only the last chunk's copy is
exposed.

    pipe = HostPipeline(chunks=4)
    out = pipe.run(app, device_graph, n_samples=N, seed=7)   # list[HostChunk]
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import DeviceRun, describe, run_device
from .graph import as_device_graph
from .sharding import worker_ranges

import os
_NO_COPY = os.environ.get("ND_PIPE_NOCOPY") == "1"  # dev: time the pipeline without D2H


@dataclass
class HostChunk:
    """Final rows of samples [sample_lo, sample_lo + n) in pinned host memory."""
    sample_lo: int
    n: int
    offsets: "object"        # torch int64 [n+1], chunk-local row offsets
    ids: "object"            # torch int32 [offsets[n]]: roots, then sampled vertices
    total_sampled: int

    def rows(self):
        off = self.offsets.numpy()
        ids = self.ids.numpy()
        return [ids[off[i]:off[i + 1]] for i in range(self.n)]


class HostPipeline:
    """Chunked device run with overlapped device->host row copies.  Pinned
    buffers are owned by the pipeline and reused across runs (sized on first
    use), so steady-state runs allocate no host memory."""

    def __init__(self, chunks: int = 4, paradigm: str = "sp", step_cap: int = 10_000):
        self.chunks = max(1, int(chunks))
        self.paradigm = paradigm
        self.step_cap = step_cap
        self._pinned = {}
        self._copy_streams = []
        self.last_h2d_bytes = 0  # host->device bytes of the last run (roots)
        self._pending = []       # (copy-done event, device runs) of runs not waited for
        self._retired = []       # replaced pinned buffers, kept until the next wait
        self._phase = 0          # pinned buffer set of the next run (two alternate)

    def _buf(self, key, like):
        import torch
        b = self._pinned.get(key)
        if b is None or b.numel() < like.numel() or b.dtype != like.dtype:
            if b is not None:  # a copy of an earlier run may still target it
                self._retired.append(b)
            b = torch.empty(max(like.numel(), 1), dtype=like.dtype, pin_memory=True)
            self._pinned[key] = b
        return b[:like.numel()]

    def run(self, app, graph, n_samples: int, seed: int = 0, sample_lo: int = 0,
            roots_host=None) -> list:
        """Run `app` for samples [sample_lo, sample_lo + n_samples).  `roots_host`
        (optional pinned int64 [n_samples * R]) replaces the keyed default roots;
        each chunk's slice is uploaded before the chunk runs.  Returns one
        HostChunk per chunk, valid until the next run of this pipeline."""
        return self.run_jobs(graph, [(app, n_samples, seed, sample_lo, roots_host)])[0]

    def run_jobs(self, graph, jobs, wait: bool = True) -> list:
        """Several apps at once through one pipeline: job = (app, n_samples,
        seed, sample_lo, roots_host[, chunks]).  Each job runs on its own compute stream
        and host thread (engine.run_device_concurrent's scheme) with its own
        copy stream, so one job's copies and tail overlap the others' bulk;
        one synchronisation at the end.  Returns one HostChunk list per job.

        wait=False returns as soon as every chunk has sampled and its copy is
        queued, so the caller's next run samples while this run's last rows
        are still crossing PCIe; its rows are valid after `wait()`.  Runs
        alternate between two pinned buffer sets, so a run's rows stay valid
        while the next run is in flight."""
        import torch
        self._release(block=False)
        phase = self._phase
        if not wait:
            self._phase ^= 1
        from .engine import _job_pool, gpu_share, job_streams
        L = _lib.load()
        dg = as_device_graph(graph)
        k = len(jobs)
        while len(self._copy_streams) < 1:
            self._copy_streams.append(torch.cuda.Stream())
        cur = torch.cuda.current_stream()
        dev = torch.cuda.current_device()
        streams = job_streams(k)
        # every job's roots go up in one copy before any sampling starts: a
        # host->device copy running under the walk kernels slows them several
        # fold (tools/probe_copy_interference.py), device->host copies do not.
        # Jobs sharing one host roots array share its upload.
        per_chunk = os.environ.get("ND_PIPE_ROOTS") == "chunk"  # dev: the old per-chunk upload
        dev_roots, self.last_h2d_bytes = {}, 0
        if not per_chunk:
            with torch.cuda.stream(cur):
                for job in jobs:
                    rh = job[4]
                    if rh is not None and id(rh) not in dev_roots:
                        dev_roots[id(rh)] = rh.to("cuda", non_blocking=True)
                        self.last_h2d_bytes += rh.numel() * rh.element_size()
        for st in streams:
            st.wait_stream(cur)

        import threading
        first_done = threading.Event()  # job 0's first chunk: its copies start the link

        def one(ji, job, st, cs):
            app, n_samples, seed, sample_lo, roots_host = job[:5]
            chunks = job[5] if len(job) > 5 and job[5] else self.chunks
            torch.cuda.set_device(dev)
            plan = describe(app)
            if isinstance(chunks, (list, tuple)):  # relative chunk sizes
                parts = weighted_plan(n_samples, chunks)
            else:
                parts = chunk_plan(n_samples, chunks, lead=(ji == 0 and k > 1))
            out, held = [], []
            if ji > 0 and k > 1:
                first_done.wait(timeout=60)  # the link gets busy before the GPU is shared
            try:
                with gpu_share(k):
                    return _chunks(ji, app, n_samples, seed, sample_lo, roots_host, st, cs, plan,
                                   parts, out, held)
            finally:
                if ji == 0:  # job 0 without chunks (or failing) must not stall the others
                    first_done.set()

        def _chunks(ji, app, n_samples, seed, sample_lo, roots_host, st, cs, plan, parts, out,
                    held):
            with torch.cuda.stream(st):
                for ci, (lo, hi) in enumerate(parts):
                    n = hi - lo
                    if trace is not None:
                        e_c0 = torch.cuda.Event(enable_timing=True)
                        e_c0.record(st)
                    if roots_host is not None:
                        R = len(roots_host) // max(n_samples, 1)
                        if per_chunk:
                            droots = roots_host[lo * R:hi * R].to("cuda", non_blocking=True)
                            self.last_h2d_bytes += droots.numel() * droots.element_size()
                        else:
                            droots = dev_roots[id(roots_host)][lo * R:hi * R]
                        held.append(droots)
                        dr = _run_walk_with_roots(plan, dg, droots, R, sample_lo + lo, n, seed,
                                                  self.paradigm, self.step_cap)
                    else:
                        dr = run_device(app, dg, n_samples=n, sample_lo=sample_lo + lo, seed=seed,
                                        paradigm=self.paradigm, step_cap=self.step_cap, stream=st,
                                        sync=False)
                    off = dr.view(_lib.F_FINAL_OFF)
                    ids = dr.narrow_ids(stream=_lib.stream_ptr(st))
                    ready = torch.cuda.Event()
                    ready.record(st)
                    cs.wait_event(ready)
                    h_off = self._buf((phase, ji, ci, "off"), off)
                    h_ids = self._buf((phase, ji, ci, "ids"), ids)
                    if trace is not None:
                        e_d0 = torch.cuda.Event(enable_timing=True)
                        e_d0.record(cs)
                    if not _NO_COPY:  # cudaMemcpyAsync on the copy stream (nd_result_copy)
                        csp = _lib.stream_ptr(cs)
                        _lib.check(L.nd_result_copy(dr._h, _lib.F_FINAL_OFF, _lib.ptr(h_off), csp),
                                   "nd_result_copy")
                        _lib.check(L.nd_result_copy(dr._h, _lib.F_FINAL_IDS32, _lib.ptr(h_ids), csp),
                                   "nd_result_copy")
                    if trace is not None:
                        e_c1 = torch.cuda.Event(enable_timing=True)
                        e_c1.record(st)
                        e_d1 = torch.cuda.Event(enable_timing=True)
                        e_d1.record(cs)
                        trace.append((getattr(app, "name", "?"), ci, e_c0, e_c1, e_d0, e_d1,
                                      h_ids.numel() * 4))
                    held.append(dr)
                    out.append(HostChunk(sample_lo + lo, n, h_off, h_ids, dr.total_sampled))
                    if ji == 0:
                        first_done.set()
            return out, held

        trace = [] if os.environ.get("ND_PIPE_TRACE") == "1" else None
        t0 = None
        if trace is not None:
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(cur)
        # one copy stream for every job: the device has one D2H engine, so the
        # copies go out in completion order
        cs0 = self._copy_streams[0]
        futs = [_job_pool(k).submit(one, ji, job, st, cs0)
                for ji, (job, st) in enumerate(zip(jobs, streams))]
        done = [f.result() for f in futs]
        if not wait:  # the runs' buffers live until their copies are done
            ev = torch.cuda.Event()
            ev.record(cs0)
            self._pending.append((ev, [h for _, held in done for h in held]))
            return [out for out, _ in done]
        cur.wait_stream(cs0)
        cur.synchronize()
        if trace is not None:  # chunk timeline (ms from the call): compute start/end, copy end
            import sys
            for name, ci, c0, c1, d0, d1, nb in trace:
                print(f"[pipe] {name:9s} chunk {ci}: compute {t0.elapsed_time(c0):7.2f} -> "
                      f"{t0.elapsed_time(c1):7.2f}  copy {t0.elapsed_time(d0):7.2f} -> "
                      f"{t0.elapsed_time(d1):7.2f}  ({nb / 1e6:.0f} MB)", file=sys.stderr)
        for _, held in done:
            for h in held:
                if isinstance(h, DeviceRun):
                    h.close()
        self._release(block=True)
        return [out for out, _ in done]

    def wait(self) -> None:
        """Wait for every run issued with wait=False (its rows are then in
        host memory) and release its device buffers."""
        self._release(block=True)

    def _release(self, block: bool) -> None:
        keep = []
        for ev, held in self._pending:
            if block:
                ev.synchronize()
            elif not ev.query():
                keep.append((ev, held))
                continue
            for h in held:
                if isinstance(h, DeviceRun):
                    h.close()
        self._pending = keep
        if not keep:
            self._retired = []


def chunk_plan(n: int, chunks: int, lead: bool = False) -> list:
    """Contiguous sample-id chunks.  With `lead`, the first chunk is a quarter
    of the others, so its rows reach the host (and the PCIe link gets busy)
    early while the rest of the GPU work is still ahead."""
    if n <= 0:
        return []
    if chunks <= 1 or not lead:
        return [(lo, hi) for lo, hi in worker_ranges(n, chunks) if hi > lo]
    first = max(1, n // (4 * chunks - 3))
    rest = [(first + lo, first + hi) for lo, hi in worker_ranges(n - first, chunks - 1) if hi > lo]
    return [(0, first)] + rest


def weighted_plan(n: int, weights) -> list:
    """Contiguous sample-id chunks with sizes proportional to `weights`
    (e.g. (1, 4, 4, 4, 1): small first and last chunks, so the link starts
    early and the last exposed copy is short)."""
    if n <= 0:
        return []
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or len(w) == 0 or (w <= 0).any():
        raise ValueError("chunk weights must be positive")
    cuts = np.rint(np.concatenate([[0.0], np.cumsum(w)]) / w.sum() * n).astype(np.int64)
    return [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _run_walk_with_roots(plan, dg, droots, R, lo, n, seed, paradigm, step_cap) -> DeviceRun:
    """nd_run_walk with caller-uploaded roots (device int64 [n * R])."""
    import ctypes as C
    if plan.kind != "walk":
        raise ValueError("explicit roots are supported for walk apps in the host pipeline")
    L = _lib.load()
    kp = np.ascontiguousarray(plan.kparams, dtype=np.float64)
    h = C.c_void_p()
    par = _lib.ND_TP if paradigm == "tp" else _lib.ND_SP
    _lib.check(L.nd_run_walk(dg.handle, plan.code, _lib.ptr(kp), len(kp), lo, n, _lib.ptr(droots), R,
                             C.c_uint64(seed & (2**64 - 1)), plan.steps, step_cap, par,
                             _lib.stream_ptr(), C.byref(h)), "nd_run_walk")
    return DeviceRun(h, plan, dg, paradigm, lo, 0.0)

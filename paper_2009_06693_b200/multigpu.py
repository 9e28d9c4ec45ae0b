"""Sample-sharded multi-GPU runs (bench.py:123-153 of the
reference).

One process per GPU.  The graph is replicated (each rank regenerates the same
keyed graph or uploads the same arrays); sample ids are split by
``worker_ranges`` and each rank runs its contiguous range with the global ids,
so the concatenated rows are byte-identical to a single-GPU run.  The only
collective is the final gather of the compacted rows to rank 0: an
``all_gather`` of the per-rank sizes, then point-to-point sends of each
rank's exact row bytes straight into their place in rank 0's output (NCCL
over NVLink on GPUs, gloo on CPU tensors in the tests; no padding, no
concatenation copy).
"""

from __future__ import annotations

import numpy as np

from .sharding import piece_ranges, shard_for_rank, worker_ranges  # noqa: F401


def gather_rows(off, ids, group=None, dst: int = 0):
    """Gather per-rank final-layout CSR pieces (off[n_r+1], ids) to `dst`.

    Works for any torch.distributed backend; tensors live on the backend's
    device (CUDA for NCCL, CPU for gloo).  `ids` may be int64 (F_FINAL_IDS) or
    int32 (F_FINAL_IDS32, half the NVLink bytes).  Returns (off, ids) concatenated in
    rank order on `dst` (None elsewhere).  On NCCL the transfers are queued
    on the communicator's stream, ordered after the caller's current stream;
    the returned tensors are ready for the caller's current stream."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "gloo" and ids.is_cuda:
        off, ids = off.cpu(), ids.cpu()  # gloo moves host tensors
    dev = ids.device
    sizes = torch.tensor([off.numel() - 1, ids.numel()], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(ws)]
    dist.all_gather(all_sizes, sizes, group=group)
    ns = [int(s[0]) for s in all_sizes]
    es = [int(s[1]) for s in all_sizes]
    peer = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    ops = []
    if rank != dst:
        if ns[rank] > 0:  # offsets without the leading 0, then the ids
            ops.append(dist.P2POp(dist.isend, off[1:].contiguous(), peer(dst), group))
        if es[rank] > 0:
            ops.append(dist.P2POp(dist.isend, ids.contiguous(), peer(dst), group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return None, None
    out_off = torch.empty(sum(ns) + 1, dtype=torch.int64, device=dev)
    out_ids = torch.empty(sum(es), dtype=ids.dtype, device=dev)
    out_off[:1] = 0
    n0, e0, bases = 0, 0, []
    for r in range(ws):
        o_sl = out_off[1 + n0:1 + n0 + ns[r]]
        i_sl = out_ids[e0:e0 + es[r]]
        if r == rank:
            o_sl.copy_(off[1:])
            i_sl.copy_(ids)
        else:
            if ns[r] > 0:
                ops.append(dist.P2POp(dist.irecv, o_sl, peer(r), group))
            if es[r] > 0:
                ops.append(dist.P2POp(dist.irecv, i_sl, peer(r), group))
        bases.append((o_sl, e0))
        n0 += ns[r]
        e0 += es[r]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for o_sl, base in bases:  # rank-local offsets -> global
        if base and o_sl.numel():
            o_sl += base
    return out_off, out_ids


def run_sharded(app, graph, n_samples: int, seed: int, paradigm: str = "sp", group=None):
    """This rank's share of an N-sample job on its GPU, gathered to rank 0.
    Returns (final_off, final_ids int32) on rank 0, (None, None) elsewhere."""
    import torch.distributed as dist
    from . import _lib
    from .engine import run_device
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_for_rank(n_samples, ws, rank)
    dr = run_device(app, graph, n_samples=hi - lo, sample_lo=lo, seed=seed, paradigm=paradigm)
    off, ids = gather_rows(dr.view(_lib.F_FINAL_OFF), dr.narrow_ids(), group)
    if off is not None:
        off, ids = off.clone(), ids.clone()
    dr.close()
    return off, ids


class ShardedJob:
    """A whole multi-app sampling job split over the ranks of `group`, through
    the public API end to end (bench.py:123-153 +
    driver.py:175-186 of the reference): every rank holds the replicated
    graph and runs its ``worker_ranges`` share of each app's sample ids.

    Per ``run()``: each rank uploads its shards' roots from pinned host memory
    and samples every app concurrently (one stream and host thread per app).
    An app's shard may be cut into ``chunks`` contiguous pieces run one after
    another on its stream; each piece's compacted rows go to `dst` over NCCL
    as soon as it is done (the gather of one piece overlaps the sampling of
    the next and of the other apps), and `dst` copies them into pinned host
    buffers on a copy stream (``to_host``).  The rows on `dst` equal one
    single-GPU run of the whole job, piece by piece.

    jobs: list of (app, n_samples_total, seed[, chunks]).  Roots are the keyed
    defaults (apps.py:83-103), produced once at construction into pinned
    memory."""

    def __init__(self, graph, jobs, group=None, dst: int = 0, paradigm: str = "sp",
                 to_host: bool = True):
        import ctypes as C
        import torch
        import torch.distributed as dist
        from . import _lib
        from .engine import describe
        from .graph import as_device_graph
        self.dg = as_device_graph(graph)
        self.group, self.dst, self.paradigm, self.to_host = group, dst, paradigm, to_host
        self.dist = dist.is_available() and dist.is_initialized()
        ws = dist.get_world_size(group) if self.dist else 1
        rank = dist.get_rank(group) if self.dist else 0
        self.rank, self.ws = rank, ws
        self.jobs = []
        L = _lib.load()
        for job in jobs:
            app, n_total, seed = job[:3]
            chunks = max(1, int(job[3])) if len(job) > 3 else 1
            plan = describe(app)
            if plan.R != 1 or plan.kind == "collective":
                raise ValueError("ShardedJob runs walk and individual apps with one root per sample")
            lo, hi = shard_for_rank(n_total, ws, rank)
            n = hi - lo
            pieces = piece_ranges(n_total, ws, rank, chunks)
            droots = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
            if n:
                _lib.check(L.nd_uniform_roots(self.dg.handle, 1, C.c_uint64(seed), lo, n,
                                              _lib.ptr(droots), _lib.stream_ptr()),
                           "nd_uniform_roots")
            roots_host = droots[:n].cpu().pin_memory()
            self.jobs.append(dict(app=app, n_total=n_total, seed=seed, lo=lo, n=n,
                                  roots_host=roots_host, pieces=pieces))
        self._host = {}
        self._copy = torch.cuda.Stream()
        self.last = {}

    def _pinned(self, key, like):
        import torch
        b = self._host.get(key)
        if b is None or b.numel() < like.numel() or b.dtype != like.dtype:
            b = torch.empty(max(like.numel(), 1), dtype=like.dtype, pin_memory=True)
            self._host[key] = b
        return b[:like.numel()]

    def run(self, order=None):
        """One step.  Returns, per job (job order), the list of its pieces'
        (off, ids) on `dst` -- pinned host tensors (device tensors when
        to_host=False) valid until the next run; piece c holds every rank's
        c-th chunk in rank order; None on other ranks.  `order`: the order in
        which the jobs' pieces are gathered (the same on every rank; default
        job order).  self.last: this rank's sampled edges, H2D / D2H bytes."""
        import queue

        import torch
        from . import _lib
        from .engine import _job_pool, gpu_share, job_streams, run_device
        cur = torch.cuda.current_stream()
        dev = torch.cuda.current_device()
        h2d = 0
        droots = []
        for j in self.jobs:
            droots.append(j["roots_host"].to("cuda", non_blocking=True) if j["n"] else None)
            h2d += j["roots_host"].numel() * 8 if j["n"] else 0
        k = len(self.jobs)
        streams = job_streams(k)
        for st in streams:
            st.wait_stream(cur)
        queues = [queue.Queue() for _ in range(k)]

        def runner(i, st):
            j = self.jobs[i]
            torch.cuda.set_device(dev)
            with torch.cuda.stream(st), gpu_share(k):
                for a, b in j["pieces"]:
                    dr = None
                    try:
                        if b > a:
                            dr = run_device(j["app"], self.dg, n_samples=b - a, sample_lo=a,
                                            seed=j["seed"], paradigm=self.paradigm, stream=st,
                                            sync=False,
                                            roots_device=droots[i][a - j["lo"]:b - j["lo"]])
                    except BaseException as e:  # the main thread re-raises it in order
                        queues[i].put((e, None))
                        return
                    ev = torch.cuda.Event()
                    ev.record(st)
                    queues[i].put((dr, ev))

        futs = [_job_pool(k).submit(runner, i, st) for i, st in enumerate(streams)]
        out = [[] for _ in range(k)]
        edges, d2h, runs = 0, 0, []
        empty_off = torch.zeros(1, dtype=torch.int64, device="cuda")
        empty_ids = torch.empty(0, dtype=torch.int32, device="cuda")
        seq = [(i, c) for i in (order if order is not None else range(k))
               for c in range(len(self.jobs[i]["pieces"]))]
        for i, c in seq:
            dr, ev = queues[i].get()
            if isinstance(dr, BaseException):
                # the other jobs finish before the error propagates (no orphaned work)
                for f in futs:
                    f.exception()
                for r in runs:
                    r.close()
                raise dr
            cur.wait_event(ev)
            if dr is not None:
                runs.append(dr)
                edges += dr.total_sampled
                off, ids = dr.view(_lib.F_FINAL_OFF), dr.narrow_ids()
            else:
                off, ids = empty_off, empty_ids
            if self.dist and self.ws > 1:
                off, ids = gather_rows(off, ids, self.group, self.dst)
            if off is None:
                continue
            if self.to_host:  # rank dst: rows to pinned host memory on the copy stream
                self._copy.wait_stream(cur)
                ho, hi = self._pinned((i, c, "off"), off), self._pinned((i, c, "ids"), ids)
                with torch.cuda.stream(self._copy):
                    ho.copy_(off, non_blocking=True)
                    hi.copy_(ids, non_blocking=True)
                if off.is_cuda:
                    off.record_stream(self._copy)
                    ids.record_stream(self._copy)
                d2h += off.numel() * 8 + ids.numel() * ids.element_size()
                out[i].append((ho, hi))
            else:
                out[i].append((off.clone() if self.ws == 1 else off,
                               ids.clone() if self.ws == 1 else ids))
        for f in futs:
            f.result()
        if self.to_host:
            cur.wait_stream(self._copy)
        # a run's buffers are freed stream-ordered on its own stream: order that
        # stream after the gathers and copies (the current stream waited on them)
        for st in streams:
            st.wait_stream(cur)
        for dr in runs:
            dr.close()
        self.last = dict(edges=edges, h2d_bytes=h2d, d2h_bytes=d2h)
        return out if (not self.dist or self.ws == 1 or self.rank == self.dst) else None

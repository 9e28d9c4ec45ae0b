"""Out-of-core sub-graph shuttling.

NextDoor samples graphs larger than GPU memory by keeping the graph in host
memory and moving it to the device one sub-graph at a time, running every
sample whose transit lies in the resident sub-graph.  Here the graph's
vertices are cut into contiguous partitions whose column (and prefix) slices
fit the given device budget; the CUDA side (csrc/nd_ooc.cu) double-buffers
the slices on a copy stream and advances DeepWalk walkers / k-hop parents in
the resident partition.  Rows are identical to an in-core run of the same
job (keyed RNG), so ``tp_run``/``sp_run``/``run_device`` accept a
``ShuttledGraph`` where they accept a device graph:

    sg = ShuttledGraph.from_graph(graph, device_budget_bytes=8 << 30)
    out = tp_run(make_app("deepwalk"), sg, make_samples(app, sg, N, seed), cfg)

Shuttled apps: DeepWalk, PPR (unbounded walks up to the step cap) and
k-hop.  Every other app (node2vec reads its previous transit's row as well;
MultiRW; the collective apps) runs the ordinary sample-parallel kernels over
the same graph read in place from host memory (``ShuttledGraph.mapped()``,
zero copy), slower but with the same rows.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import UnsupportedAppError


class ShuttledGraph:
    """A CSR kept in host memory and shuttled to the device per partition.

    row_offsets int64 [V+1], col_indices (any int dtype, stored int32),
    prefix f64 [E] (the reference's sequential per-row inclusive prefix,
    graph.py:49-55) or None for unit weights."""

    def __init__(self, row_offsets, col_indices, prefix=None, *, device_budget_bytes: int,
                 register_host: bool = True, remap=None, weights=None):
        L = _lib.load()
        self._row = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self._col = np.ascontiguousarray(col_indices, dtype=np.int32)
        self._pre = None if prefix is None else np.ascontiguousarray(prefix, dtype=np.float64)
        # the weights themselves are read only by the zero-copy path (node2vec's
        # acceptance test, the collective apps)
        self._w = None if (weights is None or prefix is None) else np.ascontiguousarray(
            weights, dtype=np.float64)
        self._mapped = None
        self.n_vertices = len(self._row) - 1
        self.n_edges = len(self._col)
        if self._pre is not None and len(self._pre) != self.n_edges:
            raise ValueError("prefix must have one entry per edge")
        self.unit_weights = self._pre is None
        self._remap = remap
        h = C.c_void_p()
        _lib.check(L.nd_ooc_graph_create(_lib.ptr(self._row), _lib.ptr(self._col),
                                         _lib.ptr(self._pre), self.n_vertices, self.n_edges,
                                         int(device_budget_bytes), int(bool(register_host)),
                                         _lib.stream_ptr(), C.byref(h)), "nd_ooc_graph_create")
        self._h = h

    @classmethod
    def from_graph(cls, graph, device_budget_bytes: int, register_host: bool = True):
        """From a host Graph (this package's or the reference's): unit-weight
        graphs shuttle columns only, weighted ones columns + prefix."""
        w = np.asarray(graph.weights)
        unit = bool(np.all(w == 1.0))
        pre = None if unit else np.asarray(graph.per_vertex_weight_prefix)
        return cls(graph.row_offsets, graph.col_indices, pre, device_budget_bytes=device_budget_bytes,
                   register_host=register_host, remap=getattr(graph, "remap", None),
                   weights=None if unit else w)

    def mapped(self):
        """The same graph read in place from host memory by the ordinary
        kernels (zero copy, nd_graph_create_mapped): a DeviceGraph whose only
        device-resident arrays are the row offsets and per-row maxima.  The
        out-of-core path of every app the partition shuttle does not run."""
        if self._mapped is None:
            from .graph import DeviceGraph
            if self._pre is not None and self._w is None:
                raise UnsupportedAppError("zero-copy runs of a weighted graph need its weights "
                                          "(ShuttledGraph.from_graph keeps them)")
            h = C.c_void_p()
            _lib.check(_lib.load().nd_graph_create_mapped(
                _lib.ptr(self._row), _lib.ptr(self._col), _lib.ptr(self._w), _lib.ptr(self._pre),
                self.n_vertices, self.n_edges, _lib.stream_ptr(), C.byref(h)),
                "nd_graph_create_mapped")
            self._mapped = DeviceGraph(h, remap=self._remap)
        return self._mapped

    @property
    def handle(self):
        return self._h

    @property
    def remap(self):
        return self._remap

    def info(self) -> dict:
        """Partitions, edges per slice buffer, device bytes held, host->device
        slice bytes shuttled and slice uploads so far."""
        v = [C.c_int64() for _ in range(5)]
        _lib.check(_lib.load().nd_ooc_graph_info(self._h, *[C.byref(x) for x in v]))
        keys = ("parts", "slice_edges", "device_bytes", "bytes_shuttled", "uploads")
        return dict(zip(keys, (x.value for x in v)))

    def partitions(self) -> np.ndarray:
        """Vertex cut points [parts + 1]."""
        P = self.info()["parts"]
        out = np.zeros(P + 1, dtype=np.int64)
        _lib.check(_lib.load().nd_ooc_graph_parts(self._h, _lib.ptr(out), P + 1))
        return out

    def degree(self, v: int) -> int:
        return int(self._row[v + 1] - self._row[v])

    def close(self):
        if self._mapped is not None:
            self._mapped.close()
            self._mapped = None
        if self._h is not None and _lib._lib is not None:
            _lib._lib.nd_ooc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shuttle_supported(plan) -> bool:
    """Apps the partition shuttle runs (one resident row per step): DeepWalk,
    PPR and k-hop with fixed fanouts; everything else runs zero copy."""
    if plan.R != 1:
        return False
    if plan.kind == "walk":
        return (plan.code == 0 and plan.steps >= 0) or plan.code == 1
    return (plan.kind == "individual" and plan.code == 3 and plan.unique is None
            and len(plan.fanouts) >= 1)


def run_out_of_core(plan, sg: ShuttledGraph, lo: int, n: int, roots, seed: int, paradigm: str,
                    stream=None, step_cap: int = 10_000):
    """One job over a shuttled graph (engine.run_device dispatches here);
    returns a DeviceRun.  `roots`: host int64 [n] or None (keyed roots)."""
    import time

    import torch

    from .engine import DeviceRun
    L = _lib.load()
    droots = None
    if roots is not None:
        if plan.R != 1 or len(roots) != n:
            raise UnsupportedAppError("out-of-core runs take one root per sample")
        droots = torch.from_numpy(np.ascontiguousarray(roots, dtype=np.int64)).cuda()
    h = C.c_void_p()
    sp = _lib.stream_ptr(stream)
    t0 = time.perf_counter()
    walk = plan.kind == "walk" and plan.R == 1
    if walk and ((plan.code == 0 and plan.steps >= 0) or plan.code == 1):
        # DeepWalk: its walk length; PPR: unbounded walks up to the step cap
        kp = np.ascontiguousarray(plan.kparams, dtype=np.float64)
        steps = plan.steps if plan.code == 0 else (min(plan.steps, step_cap) if plan.steps >= 0
                                                   else step_cap)
        _lib.check(L.nd_run_walk_ooc(sg.handle, plan.code, _lib.ptr(kp), len(kp), lo, n,
                                     _lib.ptr(droots), C.c_uint64(seed & (2**64 - 1)), steps,
                                     sp, C.byref(h)), "nd_run_walk_ooc")
    elif (plan.kind == "individual" and plan.code == 3 and plan.R == 1 and plan.unique is None
          and len(plan.fanouts) >= 1):
        fan = np.ascontiguousarray(plan.fanouts, dtype=np.int64)
        _lib.check(L.nd_run_individual_ooc(sg.handle, plan.code, _lib.ptr(fan), len(fan), lo, n,
                                           _lib.ptr(droots), C.c_uint64(seed & (2**64 - 1)), sp,
                                           C.byref(h)), "nd_run_individual_ooc")
    else:
        raise UnsupportedAppError(f"app {plan.name!r} is not shuttled (engine.run_device runs "
                                  "it zero copy over ShuttledGraph.mapped())")
    torch.cuda.synchronize()
    return DeviceRun(h, plan, sg, paradigm, lo, time.perf_counter() - t0)

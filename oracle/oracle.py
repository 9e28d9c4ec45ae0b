"""ctypes front-end of the C oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product package never does.  It restates the
reference trawl algorithm in C (``oracle/nd_oracle.c``) and exposes it with
numpy arrays.  Its outputs are pinned against the reference's own
known-answer values and golden hashes in ``tests/golden/`` (see
``tests/test_oracle.py``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libndoracle.so")

NULL_VERTEX = -1
K_DEEPWALK, K_PPR, K_NODE2VEC, K_KHOP, K_MULTIRW = range(5)
C_LAYER, C_IMPORTANCE, C_MVS, C_CLUSTERGCN = range(4)
ERR_STALL, ERR_APP, ERR_ARG, ERR_NOMEM = 1, 2, 3, 4


class OracleStallError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, OpenMP) into oracle/_build/."""
    src = os.path.join(HERE, "nd_oracle.c")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src),
                                                  os.path.getmtime(os.path.join(HERE, "nd_oracle.h")))):
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared",
                           "-ffp-contract=off", src, "-o", LIB_PATH])
    return LIB_PATH


_lib = None
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.ndo_key_u64.restype = C.c_uint64
        L.ndo_key_u64.argtypes = [C.c_uint64] + [C.c_int64] * 6
        L.ndo_key_uniform.restype = C.c_double
        L.ndo_key_uniform.argtypes = [C.c_uint64] + [C.c_int64] * 6
        L.ndo_cluster_roots.restype = C.c_int64
        L.ndo_transit_schedule.restype = C.c_int64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _take(ptr, n, dtype=np.int64):
    """Copy a malloc'd C array into numpy and free it."""
    if n:
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_int64)), shape=(n,)).astype(dtype, copy=True)
    else:
        arr = np.empty(0, dtype=dtype)
    lib().ndo_free(ptr)
    return arr


def _c64(a, dtype=np.int64):
    return np.ascontiguousarray(a, dtype=dtype)


@dataclass
class OGraph:
    """CSR arrays with the reference Graph's field meanings (graph.py:36-55)."""
    n_vertices: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    weights: np.ndarray
    per_vertex_weight_prefix: np.ndarray
    per_vertex_max_weight: np.ndarray
    remap: np.ndarray

    @property
    def n_edges(self):
        return len(self.col_indices)


def make_graph(row_offsets, col_indices, weights=None, remap=None) -> OGraph:
    row = _c64(row_offsets)
    col = _c64(col_indices)
    V = len(row) - 1
    w = _c64(np.ones(len(col)) if weights is None else weights, np.float64)
    pre = segmented_prefix_sum(w, row)
    mx = segment_max(w, row)
    rm = np.arange(V, dtype=np.int64) if remap is None else _c64(remap)
    return OGraph(V, row, col, w, pre, mx, rm)


def key_u64(seed, sample_id=0, step=0, transit_idx=0, slot=0, domain=0, draw=0) -> int:
    return int(lib().ndo_key_u64(seed & (2**64 - 1), sample_id, step, transit_idx, slot, domain, draw))


def key_uniform(seed, sample_id=0, step=0, transit_idx=0, slot=0, domain=0, draw=0) -> float:
    return float(lib().ndo_key_uniform(seed & (2**64 - 1), sample_id, step, transit_idx, slot, domain, draw))


def segmented_prefix_sum(values, offsets):
    v = _c64(values, np.float64)
    o = _c64(offsets)
    out = np.empty(len(v), dtype=np.float64)
    lib().ndo_segmented_prefix_sum(_p(v), _p(o), C.c_int64(len(o) - 1), _p(out))
    return out


def segment_max(values, offsets):
    v = _c64(values, np.float64)
    o = _c64(offsets)
    out = np.empty(len(o) - 1, dtype=np.float64)
    lib().ndo_segment_max(_p(v), _p(o), C.c_int64(len(o) - 1), _p(out))
    return out


def _check(rc):
    if rc == ERR_STALL:
        raise OracleStallError("rejection sampler exceeded 1000000 tries")
    if rc == ERR_APP:
        raise ValueError("unknown app code")
    if rc:
        raise RuntimeError(f"oracle error {rc}")


def individual_batch(app_code, params, row_offsets, col_indices, weights, weight_prefix,
                     max_weight, transits, t_prev, sample_ids, transit_idxs, slots,
                     seed, step, out):
    """_ckernels.pyx:136-271 restated; same argument order as the reference."""
    arrs = [_c64(params, np.float64), _c64(row_offsets), _c64(col_indices),
            _c64(weights, np.float64), _c64(weight_prefix, np.float64),
            _c64(max_weight, np.float64), _c64(transits), _c64(t_prev),
            _c64(sample_ids), _c64(transit_idxs), _c64(slots)]
    res = np.empty(len(arrs[6]), dtype=np.int64)
    rc = lib().ndo_individual_batch(
        C.c_int(app_code), _p(arrs[0]), C.c_int64(len(arrs[0])), *[_p(a) for a in arrs[1:]],
        C.c_int64(len(res)), C.c_uint64(seed & (2**64 - 1)), C.c_int64(step), _p(res))
    _check(rc)
    out[:] = res


def uniform_roots(n_vertices, count, seed, sample_lo, n_samples):
    out = np.empty(n_samples * count, dtype=np.int64)
    lib().ndo_uniform_roots(C.c_int64(n_vertices), C.c_int64(count), C.c_uint64(seed),
                            C.c_int64(sample_lo), C.c_int64(n_samples), _p(out))
    return out.reshape(n_samples, count)


def cluster_roots(n_vertices, clusters_per_sample, num_clusters, seed, sample_id):
    L = lib()
    cnt = L.ndo_cluster_roots(C.c_int64(n_vertices), C.c_int64(clusters_per_sample),
                              C.c_int64(num_clusters), C.c_uint64(seed), C.c_int64(sample_id), None)
    out = np.empty(cnt, dtype=np.int64)
    L.ndo_cluster_roots(C.c_int64(n_vertices), C.c_int64(clusters_per_sample),
                        C.c_int64(num_clusters), C.c_uint64(seed), C.c_int64(sample_id), _p(out))
    return out


def run_chain(g: OGraph, app_code, params, roots, seed, steps, step_cap=10_000,
              paradigm="tp", n_threads=1, sample_lo=0):
    """chain.py:64-179.  roots: (n, R) int64, mutated copy returned."""
    roots = np.array(roots, dtype=np.int64, copy=True, order="C")
    n, R = roots.shape
    prm = _c64(params, np.float64)
    chain_len = np.empty(n, dtype=np.int64)
    vals_p = C.c_void_p()
    stats_p = C.c_void_p()
    n_steps = C.c_int64()
    rc = lib().ndo_run_chain(
        _p(g.row_offsets), _p(g.col_indices), _p(g.weights), _p(g.per_vertex_weight_prefix),
        _p(g.per_vertex_max_weight), C.c_int64(g.n_vertices), C.c_int(app_code), _p(prm),
        C.c_int64(len(prm)), C.c_int64(sample_lo), C.c_int64(n), _p(roots), C.c_int64(R),
        C.c_uint64(seed & (2**64 - 1)), C.c_int64(-1 if steps is None else steps),
        C.c_int64(step_cap), C.c_int(1 if paradigm == "tp" else 0), C.c_int(n_threads),
        _p(chain_len), C.byref(vals_p), C.byref(n_steps), C.byref(stats_p))
    total = int(chain_len.sum())
    vals = _take(vals_p, total)
    stats = _take(stats_p, 4 * n_steps.value).reshape(-1, 4)
    _check(rc)
    return dict(roots=roots, chain_len=chain_len, chain_vals=vals,
                n_steps=n_steps.value, stats=stats)


def _mask(unique):
    if unique is None:
        return None, 0
    m = np.ascontiguousarray(np.asarray(unique, dtype=np.uint8))
    return m, len(m)


def run_individual(g: OGraph, app_code, params, fanouts, roots_list, seed, steps,
                   step_cap=10_000, root_pick=False, needs_prev2=False,
                   paradigm="tp", sample_lo=0, unique=None):
    """driver.py:203-235 run loop with StepPlan semantics (generic path)."""
    n = len(roots_list)
    roots_off = np.zeros(n + 1, dtype=np.int64)
    roots_off[1:] = np.cumsum([len(r) for r in roots_list])
    roots = _c64(np.concatenate(roots_list) if n else np.empty(0))
    fan = _c64(fanouts)
    prm = _c64(params, np.float64)
    n_steps = C.c_int64()
    cnt_p, vals_p, stats_p = C.c_void_p(), C.c_void_p(), C.c_void_p()
    n_vals = C.c_int64()
    um, nm = _mask(unique)
    rc = lib().ndo_run_individual(
        _p(g.row_offsets), _p(g.col_indices), _p(g.weights), _p(g.per_vertex_weight_prefix),
        _p(g.per_vertex_max_weight), C.c_int64(g.n_vertices), C.c_int(app_code), _p(prm),
        C.c_int64(len(prm)), _p(fan), C.c_int64(len(fan)), C.c_int(int(root_pick)),
        C.c_int(int(needs_prev2)), C.c_int64(sample_lo), C.c_int64(n), _p(roots_off),
        _p(roots), C.c_uint64(seed & (2**64 - 1)), C.c_int64(-1 if steps is None else steps),
        C.c_int64(step_cap), C.c_int(1 if paradigm == "tp" else 0),
        _p(um) if um is not None else None, C.c_int64(nm), C.byref(n_steps),
        C.byref(cnt_p), C.byref(vals_p), C.byref(n_vals), C.byref(stats_p))
    S = n_steps.value
    counts = _take(cnt_p, S * n).reshape(S, n)
    vals = _take(vals_p, n_vals.value)
    stats = _take(stats_p, 4 * S).reshape(-1, 4)
    _check(rc)
    final_roots = [roots[roots_off[i]:roots_off[i + 1]] for i in range(n)]
    return dict(n_steps=S, step_counts=counts, vals=vals, stats=stats, roots=final_roots)


def run_collective(g: OGraph, kind, step_size, roots_list, seed, steps, max_size=0,
                   distribution=0, step_cap=10_000, sample_lo=0, unique=None):
    n = len(roots_list)
    roots_off = np.zeros(n + 1, dtype=np.int64)
    roots_off[1:] = np.cumsum([len(r) for r in roots_list])
    roots = _c64(np.concatenate(roots_list) if n else np.empty(0))
    n_steps = C.c_int64()
    ptrs = [C.c_void_p() for _ in range(6)]
    n_vals, n_rec = C.c_int64(), C.c_int64()
    um, nm = _mask(unique)
    rc = lib().ndo_run_collective(
        _p(g.row_offsets), _p(g.col_indices), C.c_int64(g.n_vertices), C.c_int(kind),
        C.c_int64(step_size), C.c_int64(max_size), C.c_int(distribution),
        C.c_int64(sample_lo), C.c_int64(n), _p(roots_off), _p(roots),
        C.c_uint64(seed & (2**64 - 1)), C.c_int64(-1 if steps is None else steps),
        C.c_int64(step_cap), _p(um) if um is not None else None, C.c_int64(nm),
        C.byref(n_steps), C.byref(ptrs[0]), C.byref(ptrs[1]),
        C.byref(n_vals), C.byref(ptrs[2]), C.byref(ptrs[3]), C.byref(ptrs[4]),
        C.byref(n_rec), C.byref(ptrs[5]))
    S = n_steps.value
    counts = _take(ptrs[0], S * n).reshape(S, n)
    vals = _take(ptrs[1], n_vals.value)
    rec_counts = _take(ptrs[2], S * n).reshape(S, n)
    rec_t = _take(ptrs[3], n_rec.value)
    rec_v = _take(ptrs[4], n_rec.value)
    stats = _take(ptrs[5], 4 * S).reshape(-1, 4)
    _check(rc)
    return dict(n_steps=S, step_counts=counts, vals=vals, rec_counts=rec_counts,
                rec_t=rec_t, rec_v=rec_v, stats=stats,
                roots=[roots[roots_off[i]:roots_off[i + 1]] for i in range(n)])


def transit_schedule(pair_transit, m):
    """build_transit_map + partition_work_classes; returns dict of arrays."""
    pt = _c64(pair_transit)
    n = len(pt)
    order = np.empty(n, dtype=np.int64)
    gs = np.empty(n + 1, dtype=np.int64)
    gt = np.empty(max(n, 1), dtype=np.int64)
    gc = np.empty(max(n, 1), dtype=np.int32)
    si = np.empty(max(n, 1), dtype=np.int64)
    G = lib().ndo_transit_schedule(_p(pt), C.c_int64(n), C.c_int64(m), _p(order), _p(gs),
                                   _p(gt), _p(gc), _p(si))
    return dict(order=order, group_start=gs[:G + 1], group_transit=gt[:G],
                group_class=gc[:G], sched_index=si[:G])


def rmat_thresholds(a=0.57, b=0.19, c=0.19):
    return int(a * 65536), int((a + b) * 65536), int((a + b + c) * 65536)


def rmat_edges(scale, n_edges, seed=0, undirected=False, weighted=True, abc=(0.57, 0.19, 0.19)):
    ta, tab, tabc = rmat_thresholds(*abc)
    m = n_edges * (2 if undirected else 1)
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    w = np.empty(m, dtype=np.float64)
    lib().ndo_rmat_edges(C.c_int(scale), C.c_int64(n_edges), C.c_uint32(ta), C.c_uint32(tab),
                         C.c_uint32(tabc), C.c_uint64(seed), C.c_int(int(undirected)),
                         C.c_int(int(weighted)), _p(src), _p(dst), _p(w))
    return src, dst, w


def from_edges(src, dst, weights, n_vertices):
    src, dst = _c64(src), _c64(dst)
    w = _c64(weights, np.float64) if weights is not None else np.ones(len(src))
    row = np.empty(n_vertices + 1, dtype=np.int64)
    col = np.empty(len(src), dtype=np.int64)
    wo = np.empty(len(src), dtype=np.float64)
    rc = lib().ndo_from_edges(_p(src), _p(dst), _p(w), C.c_int64(len(src)),
                              C.c_int64(n_vertices), _p(row), _p(col), _p(wo))
    _check(rc)
    return make_graph(row, col, wo)


def rmat_graph(scale, edge_factor=16, seed=0, undirected=False, weighted=True):
    V = 1 << scale
    src, dst, w = rmat_edges(scale, V * edge_factor, seed, undirected, weighted)
    return from_edges(src, dst, w, V)

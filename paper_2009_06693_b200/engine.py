"""Engine entry points: ``tp_run`` / ``sp_run`` (transit_parallel.py:249-257,
sample_parallel.py:102-110) on the B200 device engine.

The reference runs a Python step loop over numpy work items; here one call
hands the whole run to the device (include/nextdoor_b200.h):

  chain walks (DeepWalk, PPR, node2vec, MultiRW)  -> nd_run_walk
  multi-slot individual apps (k-hop)              -> nd_run_individual
  collective apps (layer, FastGCN/LADIES, MVS, ClusterGCN) -> nd_run_collective

``paradigm`` "tp" runs the transit-parallel scheduler (per-step radix sort of
(transit, sample) pairs, three work classes, sub-warp / CTA / grid kernels
with shared-memory-staged adjacency); "sp" runs the flat sample-parallel
kernels.  Outputs are identical (keyed RNG), as in the reference.
"""

from __future__ import annotations

import ctypes as C
import math
import time
import warnings
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .core import DEFAULT_STEP_CAP, INF_STEPS, Sample
from .errors import UnsupportedAppError
from .graph import DeviceGraph, as_device_graph, device_view
from .output import SampleSetOutput

COLLECTIVE_KINDS = {"layer": 0, "fastgcn": 1, "ladies": 1, "mvs": 2, "clustergcn": 3}


@dataclass
class EngineConfig:
    """driver.py:33-38 plus the device paradigm knob."""
    seed: int = 0
    n_workers: int = 1
    step_cap: int = DEFAULT_STEP_CAP
    use_kernels: bool = True
    paradigm: Optional[str] = None   # None: taken from tp_run / sp_run
    step_timing: bool = False        # event-time every step (RunStats.timings build_s/sample_s)


@dataclass
class StepTiming:
    step: int
    build_s: float = 0.0
    sample_s: float = 0.0
    groups_small: int = 0
    groups_medium: int = 0
    groups_large: int = 0


@dataclass
class RunStats:
    """driver.py:51-77: per-step group classes, adjacency fetches, timings."""
    paradigm: str
    n_samples: int
    timings: list = field(default_factory=list)
    adjacency_fetches: int = 0
    total_s: float = 0.0
    build_total_s: float = 0.0
    sample_total_s: float = 0.0
    compact_total_s: float = 0.0
    counters: dict = field(default_factory=dict)

    @property
    def build_s(self) -> float:
        return self.build_total_s

    @property
    def sample_s(self) -> float:
        return self.sample_total_s

    @property
    def n_steps(self) -> int:
        return len(self.timings)

    def group_totals(self):
        return (sum(t.groups_small for t in self.timings),
                sum(t.groups_medium for t in self.timings),
                sum(t.groups_large for t in self.timings))

    def throughput(self) -> float:
        return self.n_samples / self.total_s if self.total_s > 0 else float("inf")


@dataclass
class DevicePlan:
    kind: str                 # "walk" | "individual" | "collective"
    name: str
    code: int = -1
    kparams: np.ndarray = field(default_factory=lambda: np.zeros(0))
    steps: int = -1           # -1 = INF
    R: int = 1                # roots per sample (uniform roots)
    fanouts: list = field(default_factory=list)
    ckind: int = -1
    step_size: int = 0
    max_size: int = 0
    distribution: int = 0
    cps: int = 0
    nc: int = 0
    unique: Optional[np.ndarray] = None   # uint8 per step (run loop apps only)
    roots_kind: str = "keyed"             # "keyed" | "host" (custom init_roots)


_PLANS = {}  # id(app) -> (app, plan): describe() walks app.unique over up to 4096 steps


def describe(app) -> DevicePlan:
    """Map a SamplingApp (ours or the reference's) onto a device plan: by
    kernel_code for individual apps, by name + params for collective apps.
    Plans are cached per app object (apps are immutable once built)."""
    hit = _PLANS.get(id(app))
    if hit is not None and hit[0] is app:
        return hit[1]
    plan = _describe(app)
    if len(_PLANS) > 256:
        _PLANS.clear()
    _PLANS[id(app)] = (app, plan)
    return plan


def _describe(app) -> DevicePlan:
    name = getattr(app, "name", "?")
    p = dict(getattr(app, "params", {}) or {})
    steps = -1 if app.steps == INF_STEPS or (isinstance(app.steps, float) and math.isinf(app.steps)) \
        else int(app.steps)
    n_check = 4096 if steps < 0 else max(steps, 1)
    um = np.asarray([1 if app.unique(s) else 0 for s in range(n_check)], dtype=np.uint8)
    umask = um if um.any() else None
    if getattr(app, "step_transits_fn", None) is not None:
        raise UnsupportedAppError(f"{name}: custom step_transits_fn needs a Python callback")
    code = getattr(app, "kernel_code", None)
    if code is None and name in _BUNDLED_CODES:
        code = _BUNDLED_CODES[name]  # object-mode bundled app: same draws as its kernel
    kp = np.asarray(getattr(app, "kernel_params", np.zeros(0)), dtype=np.float64)
    init = getattr(app, "init_roots", None)
    R = int(getattr(init, "count", 0) or 0)
    if len(kp) == 0 and code in (1, 2):
        kp = _default_kparams(name, p)
    if code in (0, 1, 2, 4) and getattr(app, "chain_walk", False):
        # chain walks ignore unique() like the reference's run_chain (chain.py:31-40)
        if code == 4:
            R = R or int(p.get("roots_per_sample", 100))
        return DevicePlan("walk", name, code=code, kparams=kp, steps=steps, R=R or 1,
                          roots_kind=_roots_kind(app))
    if code == 3:
        fan = [int(f) for f in p.get("fanouts", [app.sample_size(s) for s in range(max(steps, 0))])]
        return DevicePlan("individual", name, code=code, kparams=kp, steps=len(fan), R=R or 1,
                          fanouts=fan, unique=umask, roots_kind=_roots_kind(app))
    if code in (0, 1, 2, 4):
        # kernel app without chain_walk: generic run loop, one slot per step
        m = [int(app.sample_size(s)) for s in range(max(steps, 1))] if steps >= 0 else [1]
        if code == 4 or any(x != 1 for x in m) or steps < 0:
            raise UnsupportedAppError(f"{name}: unsupported individual configuration")
        return DevicePlan("walk", name, code=code, kparams=kp, steps=steps, R=R or 1,
                          roots_kind=_roots_kind(app))
    if name in COLLECTIVE_KINDS:
        ck = COLLECTIVE_KINDS[name]
        plan = DevicePlan("collective", name, ckind=ck, steps=steps, unique=umask,
                          roots_kind=_roots_kind(app))
        if ck == 0:
            plan.step_size = int(p.get("step_size", app.sample_size(0)))
            plan.max_size = int(p.get("max_size", 2000))
            plan.R = R or 1
        elif ck in (1, 2):
            plan.step_size = int(p.get("step_size", app.sample_size(0)))
            plan.R = R or int(p.get("batch_size", 64))
            plan.distribution = 1 if p.get("distribution", "uniform") == "degree_sq" else 0
        else:
            plan.step_size = 1
            plan.cps = int(p.get("clusters_per_sample", 20))
            plan.nc = int(p.get("num_clusters", 100))
        return plan
    raise UnsupportedAppError(
        f"app {name!r} has no device implementation (custom Python next_fn); the B200 "
        "engine runs the bundled apps' kernels only and has no CPU fallback")


_BUNDLED_CODES = {"deepwalk": 0, "ppr": 1, "node2vec": 2, "khop": 3, "multirw": 4}


def _default_kparams(name, p):
    if name == "ppr":
        return np.asarray([p.get("termination_probability", 0.01)], dtype=np.float64)
    if name == "node2vec":
        conv = p.get("factor_convention", "reciprocal")
        return np.asarray([p.get("p", 2.0), p.get("q", 0.5), 0.0 if conv == "reciprocal" else 1.0])
    return np.zeros(0)


def _roots_kind(app) -> str:
    """'keyed' when init_roots is one of the bundled keyed initialisers (ours or
    the reference's closures, apps.py:83-103, 340-370): the device draws the
    same roots itself.  Anything else is evaluated on the host and uploaded."""
    init = getattr(app, "init_roots", None)
    if init is None:
        return "keyed"
    from .apps import ClusterRoots, UniformRoots
    if isinstance(init, (UniformRoots, ClusterRoots)):
        return "keyed"
    qn = getattr(init, "__qualname__", "")
    if qn in ("_uniform_roots.<locals>.init", "make_clustergcn.<locals>.init"):
        return "keyed"
    return "host"


class SampleRange(Sequence):
    """Samples with contiguous global ids [lo, lo+n) whose roots are drawn on
    device by the app's keyed initialiser (make_samples, driver.py:238-250)."""

    def __init__(self, app, graph, lo: int, n: int, seed: int):
        self.app, self.graph, self.lo, self.n, self.seed = app, graph, int(lo), int(n), int(seed)

    def __len__(self):
        return self.n

    def __getitem__(self, i):
        if isinstance(i, slice):
            a, b, st = i.indices(self.n)
            if st != 1:
                raise ValueError("SampleRange slices must be contiguous")
            return SampleRange(self.app, self.graph, self.lo + a, max(0, b - a), self.seed)
        i = int(i)
        if i < 0:
            i += self.n
        if not 0 <= i < self.n:
            raise IndexError("SampleRange index out of range")
        init = self.app.init_roots
        return Sample(self.lo + i, init(self.graph, self.lo + i, self.seed), self.graph)


def make_samples(app, graph, n_samples: int, seed: int, lo: int = 0) -> SampleRange:
    return SampleRange(app, graph, lo, n_samples, seed)


def _sample_spec(samples, plan, seed):
    """(sample_lo, n, roots) for the ABI; roots None = keyed on device."""
    if isinstance(samples, SampleRange):
        if samples.seed == seed and plan.roots_kind == "keyed":
            return samples.lo, samples.n, None, None
        samples = [samples[i] for i in range(samples.n)]
    samples = list(samples)
    n = len(samples)
    if n == 0:
        return 0, 0, None, None
    ids = np.asarray([s.id for s in samples], dtype=np.int64)
    if not np.array_equal(ids, np.arange(ids[0], ids[0] + n)):
        raise ValueError("the device engine needs contiguous ascending sample ids")
    roots = [np.asarray(s.roots, dtype=np.int64) for s in samples]
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(r) for r in roots])
    return int(ids[0]), n, np.concatenate(roots), off


class DeviceRun:
    """A finished device run: owns the nd_result buffers (HBM) and exposes
    zero-copy torch views plus a host SampleSetOutput."""

    def __init__(self, handle, plan, dgraph, paradigm, sample_lo, wall_s):
        self._h = handle
        self.plan = plan
        self.graph = dgraph
        self.paradigm = paradigm
        self.sample_lo = sample_lo
        self.wall_s = wall_s
        L = _lib.load()
        n, s, ts, tr = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(L.nd_result_info(handle, C.byref(n), C.byref(s), C.byref(ts), C.byref(tr)))
        self.n_samples, self.n_steps = n.value, s.value
        self.total_sampled, self.total_recorded = ts.value, tr.value
        ctr = (C.c_int64 * 12)()
        L.nd_result_counters(handle, ctr, 12)
        self.counters = dict(zip(["items", "pairs", "n2v_tries", "n2v_probes", "search",
                                  "pair_bytes", "slot_bytes", "steps", "launches", "rand_sectors",
                                  "tp_staged", "tp_inplace"],
                                 list(ctr)))
        prof = (C.c_double * 4)()
        L.nd_result_profile(handle, prof, 4)
        self.profile_ms = list(prof)
        k = C.c_int64()
        L.nd_result_step_times(handle, None, None, 0, C.byref(k))
        bt, st = (C.c_double * max(k.value, 1))(), (C.c_double * max(k.value, 1))()
        if k.value:
            L.nd_result_step_times(handle, bt, st, k.value, C.byref(k))
        self.step_ms = [(bt[i], st[i]) for i in range(k.value)]  # (build, sample) per step

    def field_count(self, f):
        p, c = C.c_void_p(), C.c_int64()
        _lib.check(_lib.load().nd_result_field(self._h, f, C.byref(p), C.byref(c)))
        return p.value, c.value

    def narrow_ids(self, stream=None):
        """Produce F_FINAL_IDS32 (int32 final ids) on device; returns its view."""
        _lib.check(_lib.load().nd_result_narrow_ids(
            self._h, _lib.stream_ptr() if stream is None else stream), "nd_result_narrow_ids")
        return self.view(_lib.F_FINAL_IDS32)

    def final_samples(self, width: int | None = None):
        """getFinalSamples (frontend/src/index.ts:160-171) without leaving the
        GPU: an int32 CUDA tensor [n_samples, width], row i = sample i's roots
        then its sampled vertices, padded with -1 (width: the longest row by
        default).  Share it zero-copy with torch.utils.dlpack.to_dlpack."""
        torch = _lib.require_cuda()
        L = _lib.load()
        if width is None:
            w = C.c_int64()
            _lib.check(L.nd_result_max_row(self._h, C.byref(w)), "nd_result_max_row")
            width = w.value
        out = torch.empty((self.n_samples, int(width)), dtype=torch.int32, device="cuda")
        _lib.check(L.nd_result_dense(self._h, int(width), _lib.ptr(out), _lib.stream_ptr()),
                   "nd_result_dense")
        return out

    def view(self, f):
        p, c = self.field_count(f)
        return None if not p else device_view(p, c, _lib.FIELD_DTYPE.get(f, "int64"), self)

    def host(self, f):
        p, c = self.field_count(f)
        if not p:
            return None
        out = np.empty(c, dtype=np.dtype(_lib.FIELD_DTYPE.get(f, "int64")))
        _lib.check(_lib.load().nd_result_copy(self._h, f, _lib.ptr(out), None))
        return out

    def stats(self) -> RunStats:
        st = self.host(_lib.F_STATS)
        st = np.zeros((0, 4), dtype=np.int64) if st is None else st.reshape(-1, 4)
        rs = RunStats(paradigm=self.paradigm, n_samples=self.n_samples, total_s=self.wall_s)
        for i, row in enumerate(st):
            b_ms, s_ms = self.step_ms[i] if i < len(self.step_ms) else (0.0, 0.0)
            rs.timings.append(StepTiming(step=i, build_s=b_ms / 1e3, sample_s=s_ms / 1e3,
                                         groups_small=int(row[0]),
                                         groups_medium=int(row[1]), groups_large=int(row[2])))
        rs.adjacency_fetches = int(st[:, 3].sum()) if len(st) else 0
        rs.build_total_s, rs.sample_total_s, rs.compact_total_s = (x / 1e3 for x in self.profile_ms[:3])
        rs.counters = dict(self.counters)
        if self.paradigm == "sp":
            for t in rs.timings:
                t.groups_small = t.groups_medium = t.groups_large = 0
        return rs

    def to_output(self, remap=None) -> SampleSetOutput:
        n = self.n_samples
        ids = np.arange(self.sample_lo, self.sample_lo + n, dtype=np.int64)
        stats = self.stats()
        final_off, final_ids = self.host(_lib.F_FINAL_OFF), self.host(_lib.F_FINAL_IDS)
        if final_ids is None:
            final_ids = np.empty(0, dtype=np.int64)
        roots = self.host(_lib.F_ROOTS)
        roots = np.empty(0, dtype=np.int64) if roots is None else roots
        if self.plan.kind == "walk":
            R = len(roots) // n if n else self.plan.R
            roots_off = np.arange(n + 1, dtype=np.int64) * R
            clen = self.host(_lib.F_CHAIN_LEN)
            clen = np.zeros(n, dtype=np.int64) if clen is None else clen
            chain = self.host(_lib.F_CHAIN_VALS)
            if chain is None:
                # non-root-pick chains: final row tail + a NULL at the death step
                nnz = np.diff(final_off) - R
                coff = np.zeros(n + 1, dtype=np.int64)
                np.cumsum(clen, out=coff[1:])
                chain = np.full(coff[-1], -1, dtype=np.int64)
                owner = np.repeat(np.arange(n), nnz)
                rank = np.arange(len(owner)) - np.repeat(np.cumsum(nnz) - nnz, nnz)
                vals_pos = (final_off[:-1] + R)[owner] + rank
                chain[coff[:-1][owner] + rank] = final_ids[vals_pos]
            else:
                coff = np.zeros(n + 1, dtype=np.int64)
                np.cumsum(clen, out=coff[1:])
            return SampleSetOutput(ids, roots_off, roots, self.n_steps, remap=remap, stats=stats,
                                   chain_off=coff, chain_vals=chain, final_off=final_off,
                                   final_ids=final_ids)
        roots_off = self.host(_lib.F_ROOTS_OFF)
        S = self.n_steps
        cnt = self.host(_lib.F_STEP_COUNTS)
        cnt = np.zeros((S, n), dtype=np.int64) if cnt is None else cnt.reshape(S, n)
        vals = self.host(_lib.F_STEP_VALS)
        rec = {}
        if self.plan.kind == "collective" and self.plan.ckind != 0:
            rc = self.host(_lib.F_REC_COUNTS)
            rec = dict(rec_counts=(np.zeros((S, n), np.int64) if rc is None else rc.reshape(S, n)),
                       rec_t=self.host(_lib.F_REC_T), rec_v=self.host(_lib.F_REC_V))
            for k in ("rec_t", "rec_v"):
                if rec[k] is None:
                    rec[k] = np.empty(0, dtype=np.int64)
        return SampleSetOutput(ids, roots_off, roots, S, remap=remap, stats=stats,
                               step_counts=cnt,
                               step_vals=np.empty(0, np.int64) if vals is None else vals,
                               final_off=final_off, final_ids=final_ids, **rec)

    def close(self):
        if self._h is not None and _lib._lib is not None:
            _lib._lib.nd_result_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_device(app, graph, samples=None, *, seed: int = 0, paradigm: str = "tp",
               step_cap: int = DEFAULT_STEP_CAP, n_samples: int | None = None,
               sample_lo: int = 0, stream=None, sync: bool = True,
               roots_device=None) -> DeviceRun:
    """Run a whole sampling job on the device; outputs stay in HBM.

    `roots_device` (walk and individual apps): a device int64 tensor
    [n_samples * R] of caller-uploaded roots for samples [sample_lo,
    sample_lo + n_samples), used in place of the keyed default roots."""
    torch = _lib.require_cuda()
    L = _lib.load()
    plan = describe(app)
    from .outofcore import ShuttledGraph, run_out_of_core, shuttle_supported
    if isinstance(graph, ShuttledGraph):  # graph in host memory, shuttled per partition
        if not shuttle_supported(plan):  # read in place over the host link instead
            return run_device(app, graph.mapped(), samples, seed=seed, paradigm="sp",
                              step_cap=step_cap, n_samples=n_samples, sample_lo=sample_lo,
                              stream=stream, sync=sync, roots_device=roots_device)
        if roots_device is not None:
            raise ValueError("roots_device is for device-resident graphs")
        if samples is None:
            samples = SampleRange(app, graph, sample_lo, n_samples or 0, seed)
        lo, n, roots, _ = _sample_spec(samples, plan, seed)
        return run_out_of_core(plan, graph, lo, n, roots, seed, paradigm, stream, step_cap)
    dg = as_device_graph(graph)
    if roots_device is not None:
        if plan.kind == "collective":
            raise ValueError("roots_device is for walk and individual apps")
        n = int(n_samples or 0)
        if n <= 0 or roots_device.numel() % n or roots_device.dtype != torch.int64:
            raise ValueError("roots_device must be int64 [n_samples * R]")
        return _run_rooted(plan, dg, roots_device, roots_device.numel() // n, sample_lo, n, seed,
                           paradigm, step_cap, stream, sync)
    if samples is None:
        samples = SampleRange(app, graph, sample_lo, n_samples or 0, seed)
    lo, n, roots, roots_off = _sample_spec(samples, plan, seed)
    par = _lib.ND_TP if paradigm == "tp" else _lib.ND_SP
    sp = _lib.stream_ptr(stream)
    h = C.c_void_p()
    t0 = time.perf_counter()
    if plan.kind == "walk":
        droots = None
        if roots is not None:
            R = int(roots_off[1] - roots_off[0]) if n else plan.R
            if not np.all(np.diff(roots_off) == R):
                raise ValueError("walk apps need the same root count for every sample")
            droots = torch.from_numpy(roots).cuda()
        else:
            R = plan.R
        kp = np.ascontiguousarray(plan.kparams, dtype=np.float64)
        rc = L.nd_run_walk(dg.handle, plan.code, _lib.ptr(kp), len(kp), lo, n, _lib.ptr(droots), R,
                           C.c_uint64(seed & (2**64 - 1)), plan.steps, step_cap, par, sp,
                           C.byref(h))
        _lib.check(rc, "nd_run_walk")
    elif plan.kind == "individual":
        droots = None
        R = plan.R
        if roots is not None:
            R = int(roots_off[1] - roots_off[0]) if n else R
            if not np.all(np.diff(roots_off) == R):
                raise ValueError("individual apps need the same root count for every sample")
            droots = torch.from_numpy(roots).cuda()
        kp = np.ascontiguousarray(plan.kparams, dtype=np.float64)
        fan = np.ascontiguousarray(plan.fanouts, dtype=np.int64)
        um = None if plan.unique is None else np.ascontiguousarray(plan.unique)
        rc = L.nd_run_individual(dg.handle, plan.code, _lib.ptr(kp), len(kp), _lib.ptr(fan),
                                 len(fan), lo, n, _lib.ptr(droots), R,
                                 C.c_uint64(seed & (2**64 - 1)), step_cap, par, _lib.ptr(um),
                                 0 if um is None else len(um), sp, C.byref(h))
        _lib.check(rc, "nd_run_individual")
    else:
        droff = dro = None
        if roots is not None:
            droff = torch.from_numpy(roots_off).cuda()
            dro = torch.from_numpy(roots).cuda()
        um = None if plan.unique is None else np.ascontiguousarray(plan.unique)
        rc = L.nd_run_collective(dg.handle, plan.ckind, plan.step_size, plan.max_size,
                                 plan.distribution, plan.steps, plan.R, plan.cps, plan.nc, lo, n,
                                 _lib.ptr(droff), _lib.ptr(dro), C.c_uint64(seed & (2**64 - 1)),
                                 step_cap, _lib.ptr(um), 0 if um is None else len(um), sp,
                                 C.byref(h))
        _lib.check(rc, "nd_run_collective")
    if sync:
        torch.cuda.synchronize()
    return DeviceRun(h, plan, dg, paradigm, lo, time.perf_counter() - t0)


def _run_rooted(plan, dg, droots, R, lo, n, seed, paradigm, step_cap, stream, sync) -> DeviceRun:
    """nd_run_walk / nd_run_individual with caller-uploaded device roots."""
    import torch
    L = _lib.load()
    kp = np.ascontiguousarray(plan.kparams, dtype=np.float64)
    par = _lib.ND_TP if paradigm == "tp" else _lib.ND_SP
    sp = _lib.stream_ptr(stream)
    h = C.c_void_p()
    t0 = time.perf_counter()
    if plan.kind == "walk":
        _lib.check(L.nd_run_walk(dg.handle, plan.code, _lib.ptr(kp), len(kp), lo, n, _lib.ptr(droots),
                                 R, C.c_uint64(seed & (2**64 - 1)), plan.steps, step_cap, par, sp,
                                 C.byref(h)), "nd_run_walk")
    else:
        fan = np.ascontiguousarray(plan.fanouts, dtype=np.int64)
        um = None if plan.unique is None else np.ascontiguousarray(plan.unique)
        _lib.check(L.nd_run_individual(dg.handle, plan.code, _lib.ptr(kp), len(kp), _lib.ptr(fan),
                                       len(fan), lo, n, _lib.ptr(droots), R,
                                       C.c_uint64(seed & (2**64 - 1)), step_cap, par, _lib.ptr(um),
                                       0 if um is None else len(um), sp, C.byref(h)),
                   "nd_run_individual")
    if sync:
        torch.cuda.synchronize()
    return DeviceRun(h, plan, dg, paradigm, lo, time.perf_counter() - t0)


_JOB_STREAMS = []
_JOB_POOL = None


def job_streams(k: int):
    """k cached side streams (one per concurrent job)."""
    import torch
    while len(_JOB_STREAMS) < k:
        _JOB_STREAMS.append(torch.cuda.Stream())
    return _JOB_STREAMS[:k]


class gpu_share:
    """Context manager for a job's host thread: runs it starts share the GPU
    with k-1 concurrent jobs (nd_set_concurrency, thread-local).  The
    persistent walk kernels then hold 1/k of every SM's CTA slots, so the jobs
    run side by side instead of one persistent grid queueing behind another."""

    _tls = None

    def __init__(self, k: int):
        self.k = max(1, int(k))

    @classmethod
    def _state(cls):
        import threading
        if cls._tls is None:
            cls._tls = threading.local()
        return cls._tls

    def __enter__(self):
        st = self._state()
        self._prev = getattr(st, "k", 1)
        st.k = self.k
        _lib.load().nd_set_concurrency(self.k)
        return self

    def __exit__(self, *a):
        self._state().k = self._prev  # nested shares restore the enclosing one
        _lib.load().nd_set_concurrency(self._prev)


def _job_pool(k: int):
    """Persistent host threads for concurrent jobs (one per job)."""
    import concurrent.futures as cf
    global _JOB_POOL
    if _JOB_POOL is None or _JOB_POOL._max_workers < k:
        _JOB_POOL = cf.ThreadPoolExecutor(max(4, k), thread_name_prefix="nd-job")
    return _JOB_POOL


def submit_device_concurrent(jobs, graph, *, paradigm: str = "sp",
                             step_cap: int = DEFAULT_STEP_CAP) -> list:
    """Start several whole sampling jobs at once, each on its own stream and
    host thread (the C-ABI call releases the GIL); a job = dict(app=...,
    n_samples=..., sample_lo=0, seed=0).  Returns one future per job whose
    result is a finished DeviceRun (its outputs complete in HBM); a job whose
    tail leaves the GPU idle (a few long PPR walks) overlaps the others' bulk.
    Outputs are exactly those of separate run_device calls; a job may carry
    `roots_device` (run_device's caller-uploaded roots)."""
    import torch
    _lib.require_cuda()
    dg = as_device_graph(graph)
    cur = torch.cuda.current_stream()
    dev = torch.cuda.current_device()
    streams = job_streams(len(jobs))
    for st in streams:
        st.wait_stream(cur)

    def one(job, st):
        torch.cuda.set_device(dev)
        with torch.cuda.stream(st), gpu_share(len(jobs)):
            return run_device(job["app"], dg, n_samples=job["n_samples"],
                              sample_lo=job.get("sample_lo", 0), seed=job.get("seed", 0),
                              paradigm=paradigm, step_cap=step_cap, stream=st, sync=False,
                              roots_device=job.get("roots_device"))

    return [_job_pool(len(jobs)).submit(one, j, st) for j, st in zip(jobs, streams)]


def run_device_concurrent(jobs, graph, *, paradigm: str = "sp",
                          step_cap: int = DEFAULT_STEP_CAP) -> list:
    """submit_device_concurrent, waited: the caller's current stream is
    ordered after every job; returns the DeviceRuns in job order."""
    import torch
    futs = submit_device_concurrent(jobs, graph, paradigm=paradigm, step_cap=step_cap)
    runs = [f.result() for f in futs]
    cur = torch.cuda.current_stream()
    for st in job_streams(len(jobs)):
        cur.wait_stream(st)
    return runs


class profiling:
    """Context manager: CUDA-event timing of every run inside it (phase totals
    in DeviceRun.profile_ms, per-step build/sample times in DeviceRun.step_ms
    and RunStats.timings; nd_set_profiling).  Process-wide switch; each
    step-structured run then records events per step and synchronises at
    its end."""

    _depth = 0

    def __enter__(self):
        if profiling._depth == 0:
            _lib.load().nd_set_profiling(1)
        profiling._depth += 1
        return self

    def __exit__(self, *a):
        profiling._depth -= 1
        if profiling._depth == 0:
            _lib.load().nd_set_profiling(0)


def _run(app, graph, samples, config, paradigm) -> SampleSetOutput:
    config = config or EngineConfig()
    # the reference's own EngineConfig (driver.py:34-40: seed, n_workers,
    # step_cap, use_kernels) is accepted as well as this package's
    par = getattr(config, "paradigm", None) or paradigm
    seed = getattr(config, "seed", 0)
    step_cap = getattr(config, "step_cap", DEFAULT_STEP_CAP)
    if getattr(config, "step_timing", False):
        with profiling():
            dr = run_device(app, graph, samples, seed=seed, paradigm=par, step_cap=step_cap)
    else:
        dr = run_device(app, graph, samples, seed=seed, paradigm=par, step_cap=step_cap)
    if dr.plan.steps < 0 and dr.n_steps >= step_cap:
        # run_chain / run_loop (chain.py:93-98, driver.py:215-220)
        warnings.warn(f"unbounded app {getattr(app, 'name', '?')!r} hit the "
                      f"{step_cap}-step cap", RuntimeWarning, stacklevel=3)
    remap = getattr(graph, "remap", None)
    if isinstance(graph, DeviceGraph):
        remap = graph.remap
    out = dr.to_output(remap=remap)
    dr.close()
    return out


def tp_run(app, graph, samples, config: EngineConfig | None = None) -> SampleSetOutput:
    """Grow every sample under transit-parallel execution on the device."""
    return _run(app, graph, samples, config, "tp")


def sp_run(app, graph, samples, config: EngineConfig | None = None) -> SampleSetOutput:
    """Sample-parallel device execution (the paper's SP baseline)."""
    return _run(app, graph, samples, config, "sp")

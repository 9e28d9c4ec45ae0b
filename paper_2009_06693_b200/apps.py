"""Bundled applications (mirror of trawl/apps.py:37-413).

``make_app(name, **overrides)`` returns a ``SamplingApp`` with the
reference's defaults (walk length 100, PPR termination 0.01, node2vec
p=2 q=0.5, k-hop fanouts [25, 10], layer 2000/1000, multi-root walks of
100 roots, batch apps 64/64, ClusterGCN 20 of 100 clusters).  Each app's
``next_fn`` documents the draw protocol the device kernels implement; it
is not evaluated on the host — the engine dispatches on ``kernel_code``
(individual apps) or ``name`` + ``params`` (collective apps).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import COLLECTIVE, INDIVIDUAL, INF_STEPS, TRANSITS_ROOT_PICK, SamplingApp
from .errors import UnsupportedAppError
from .rng import DOMAIN_CLUSTER_ASSIGN, DOMAIN_CLUSTER_PICK, DOMAIN_ROOT_INIT, key_u64

# device app codes (trawl/kernels/_pykernels.py:32-36)
K_DEEPWALK, K_PPR, K_NODE2VEC, K_KHOP, K_MULTIRW = 0, 1, 2, 3, 4
NODE2VEC_MAX_TRIES = 1_000_000  # apps.py:35

APP_NAMES = ["deepwalk", "ppr", "node2vec", "multirw", "khop", "layer",
             "fastgcn", "ladies", "clustergcn", "mvs"]


@dataclass
class Node2vecParams:   # apps.py:37-44
    p: float = 2.0
    q: float = 0.5
    walk_length: int = 100
    factor_convention: str = "reciprocal"


@dataclass
class PprParams:        # apps.py:47-49
    termination_probability: float = 0.01


@dataclass
class LayerParams:      # apps.py:52-55
    max_size: int = 2000
    step_size: int = 1000


@dataclass
class KhopParams:       # apps.py:58-60
    fanouts: list = field(default_factory=lambda: [25, 10])


@dataclass
class MultiRwParams:    # apps.py:63-66
    roots_per_sample: int = 100
    walk_length: int = 100


@dataclass
class BatchParams:      # apps.py:69-74
    batch_size: int = 64
    step_size: int = 64
    steps: int = 5
    distribution: str = "uniform"


@dataclass
class ClusterParams:    # apps.py:77-80
    clusters_per_sample: int = 20
    num_clusters: int = 100


class UniformRoots:
    """Keyed root initialiser (apps.py:83-103): ``count`` draws
    ``key_u64(seed, sid, domain=2, draw=d) % V``, distinct when V >= count.
    The device engine evaluates the same rule in ``nd_roots_kernel``."""

    def __init__(self, count: int):
        self.count = int(count)

    def __call__(self, graph, sample_id: int, seed: int) -> np.ndarray:
        V = graph.n_vertices
        roots, seen, draw = [], set(), 0
        distinct = V >= self.count
        while len(roots) < self.count:
            v = key_u64(seed, sample_id, domain=DOMAIN_ROOT_INIT, draw=draw) % V
            draw += 1
            if distinct:
                if v in seen:
                    continue
                seen.add(v)
            roots.append(v)
        return np.asarray(roots, dtype=np.int64)


class ClusterRoots:
    """ClusterGCN roots (apps.py:340-370): vertices of ``clusters_per_sample``
    keyed clusters, ascending."""

    def __init__(self, clusters_per_sample: int, num_clusters: int):
        self.clusters_per_sample = int(clusters_per_sample)
        self.num_clusters = int(num_clusters)

    def __call__(self, graph, sample_id: int, seed: int) -> np.ndarray:
        want = min(self.clusters_per_sample, self.num_clusters)
        chosen, draw = set(), 0
        while len(chosen) < want:
            chosen.add(key_u64(seed, sample_id, domain=DOMAIN_CLUSTER_PICK, draw=draw)
                       % self.num_clusters)
            draw += 1
        assign = cluster_assignment(graph, seed, self.num_clusters)
        return np.nonzero(np.isin(assign, sorted(chosen)))[0].astype(np.int64)


def cluster_assignment(graph, seed: int, num_clusters: int) -> np.ndarray:
    """vertex -> cluster id, keyed on (seed, vertex) (apps.py:340-346)."""
    from .rng import C_DOMAIN, C_DRAW, C_SAMPLE, C_SLOT, C_STEP, C_TRANSIT, MASK64, MIX_A, MIX_B
    ids = np.arange(graph.n_vertices, dtype=np.uint64)
    base = np.uint64((seed + C_STEP + C_TRANSIT + C_SLOT + C_DOMAIN * (DOMAIN_CLUSTER_ASSIGN + 1)
                      + C_DRAW) & MASK64)
    with np.errstate(over="ignore"):
        k = base + np.uint64(C_SAMPLE) * (ids + np.uint64(1))
        for _ in range(2):
            k = (k ^ (k >> np.uint64(30))) * np.uint64(MIX_A)
            k = (k ^ (k >> np.uint64(27))) * np.uint64(MIX_B)
            k = k ^ (k >> np.uint64(31))
    return (k % np.uint64(num_clusters)).astype(np.int64)


def _device_next(protocol: str):
    def next_fn(sample, transits, src_edges, step, rng):
        raise UnsupportedAppError(
            "bundled apps are evaluated by the CUDA engine (tp_run); "
            f"draw protocol: {protocol}")
    next_fn.__doc__ = protocol
    return next_fn


def make_deepwalk(walk_length: int = 100) -> SamplingApp:
    return SamplingApp(
        name="deepwalk", sampling_type=INDIVIDUAL, steps=walk_length,
        sample_size=lambda step: 1, next_fn=_device_next("draw 0 = weighted pick"),
        init_roots=UniformRoots(1), chain_walk=True, kernel_code=K_DEEPWALK,
        params={"walk_length": walk_length})


def make_ppr(params: PprParams | None = None) -> SamplingApp:
    params = params or PprParams()
    term = params.termination_probability
    return SamplingApp(
        name="ppr", sampling_type=INDIVIDUAL, steps=INF_STEPS,
        sample_size=lambda step: 1,
        next_fn=_device_next("draw 0 < term -> NULL; draw 1 = weighted pick"),
        init_roots=UniformRoots(1), chain_walk=True, kernel_code=K_PPR,
        kernel_params=np.asarray([term], dtype=np.float64),
        params={"termination_probability": term})


def node2vec_factors(params: Node2vecParams):
    """(f_ret, f_adj, f_far) per convention (apps.py:147-152)."""
    if params.factor_convention == "reciprocal":
        return 1.0 / params.p, 1.0, 1.0 / params.q
    if params.factor_convention == "direct":
        return params.p, 1.0 / params.q, 1.0
    raise ValueError(f"unknown factor convention {params.factor_convention!r}")


def make_node2vec(params: Node2vecParams | None = None) -> SamplingApp:
    params = params or Node2vecParams()
    node2vec_factors(params)  # validates the convention
    mode = 0.0 if params.factor_convention == "reciprocal" else 1.0
    return SamplingApp(
        name="node2vec", sampling_type=INDIVIDUAL, steps=params.walk_length,
        sample_size=lambda step: 1,
        next_fn=_device_next("try j: draw 2j = u % deg pick, draw 2j+1 = accept; "
                             "step 0: draw 0 = weighted pick"),
        init_roots=UniformRoots(1), needs_prev2=True, chain_walk=True,
        kernel_code=K_NODE2VEC,
        kernel_params=np.asarray([params.p, params.q, mode], dtype=np.float64),
        params={"p": params.p, "q": params.q,
                "factor_convention": params.factor_convention,
                "walk_length": params.walk_length})


def make_khop(params: KhopParams | None = None) -> SamplingApp:
    params = params or KhopParams()
    fanouts = [int(f) for f in params.fanouts]
    return SamplingApp(
        name="khop", sampling_type=INDIVIDUAL, steps=len(fanouts),
        sample_size=lambda step: fanouts[step],
        next_fn=_device_next("draw 0 = u % deg"),
        init_roots=UniformRoots(1), kernel_code=K_KHOP, params={"fanouts": fanouts})


def make_multirw(params: MultiRwParams | None = None) -> SamplingApp:
    params = params or MultiRwParams()
    return SamplingApp(
        name="multirw", sampling_type=INDIVIDUAL, steps=params.walk_length,
        sample_size=lambda step: 1,
        next_fn=_device_next("transit = roots[key(domain 1) % R]; draw 0 = u % deg; "
                             "result replaces the first equal root"),
        transit_source=TRANSITS_ROOT_PICK,
        init_roots=UniformRoots(params.roots_per_sample), chain_walk=True,
        kernel_code=K_MULTIRW,
        params={"roots_per_sample": params.roots_per_sample,
                "walk_length": params.walk_length})


def make_layer(params: LayerParams | None = None) -> SamplingApp:
    params = params or LayerParams()
    return SamplingApp(
        name="layer", sampling_type=COLLECTIVE, steps=INF_STEPS,
        sample_size=lambda step: params.step_size,
        next_fn=_device_next("take = min(m, max(0, cap - size)); slot s < take: "
                             "combined[u(slot) % n]"),
        init_roots=UniformRoots(1),
        params={"max_size": params.max_size, "step_size": params.step_size})


def make_importance(name: str, params: BatchParams | None = None) -> SamplingApp:
    params = params or BatchParams()
    if params.distribution not in ("uniform", "degree_sq"):
        raise ValueError(f"unknown distribution {params.distribution!r}")
    return SamplingApp(
        name=name, sampling_type=COLLECTIVE, steps=params.steps,
        sample_size=lambda step: params.step_size,
        next_fn=_device_next("v = u(slot) % V (or deg^2 inverse CDF); record (t, v) "
                             "for every transit t with edge t->v"),
        init_roots=UniformRoots(params.batch_size), records_edges=True,
        params={"batch_size": params.batch_size, "step_size": params.step_size,
                "steps": params.steps, "distribution": params.distribution})


def make_mvs(params: BatchParams | None = None) -> SamplingApp:
    params = params or BatchParams()
    return SamplingApp(
        name="mvs", sampling_type=COLLECTIVE, steps=1,
        sample_size=lambda step: params.step_size,
        next_fn=_device_next("i = u(slot) % n over the combined neighbourhood; "
                             "record (src_transit[i], nbr[i])"),
        init_roots=UniformRoots(params.batch_size), records_edges=True,
        params={"batch_size": params.batch_size, "step_size": params.step_size})


def make_clustergcn(params: ClusterParams | None = None) -> SamplingApp:
    params = params or ClusterParams()
    return SamplingApp(
        name="clustergcn", sampling_type=COLLECTIVE, steps=1,
        sample_size=lambda step: 1,
        next_fn=_device_next("record every combined entry whose neighbour is a root"),
        init_roots=ClusterRoots(params.clusters_per_sample, params.num_clusters),
        records_edges=True,
        params={"clusters_per_sample": params.clusters_per_sample,
                "num_clusters": params.num_clusters})


def make_app(name: str, **kwargs) -> SamplingApp:
    """Bundled app by id with parameter overrides (apps.py:389-409)."""
    if name == "deepwalk":
        return make_deepwalk(**kwargs)
    if name == "ppr":
        return make_ppr(PprParams(**kwargs) if kwargs else None)
    if name == "node2vec":
        return make_node2vec(Node2vecParams(**kwargs) if kwargs else None)
    if name == "khop":
        return make_khop(KhopParams(**kwargs) if kwargs else None)
    if name == "multirw":
        return make_multirw(MultiRwParams(**kwargs) if kwargs else None)
    if name == "layer":
        return make_layer(LayerParams(**kwargs) if kwargs else None)
    if name in ("fastgcn", "ladies"):
        return make_importance(name, BatchParams(**kwargs) if kwargs else None)
    if name == "mvs":
        return make_mvs(BatchParams(**kwargs) if kwargs else None)
    if name == "clustergcn":
        return make_clustergcn(ClusterParams(**kwargs) if kwargs else None)
    raise ValueError(f"unknown app {name!r}")

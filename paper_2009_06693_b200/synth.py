"""Synthetic input graphs (mirror of trawl/synth.py:21-113) plus the keyed
RMAT generator used for the SURVEY §8(d) C2-C5 shapes.

The small generators reproduce the reference's graphs exactly (same numpy
PCG64 draw sequence, same symmetrisation, from_edges ordering), pinned by
tests/test_synth.py against the reference-built golden graphs.  They are
inputs, not the sampling path; large graphs come from ``DeviceGraph.rmat``.
"""

from __future__ import annotations

import numpy as np

from .graph import Graph, from_edges


def _weights(n_edges, weighted, rng):
    return rng.uniform(1.0, 5.0, size=n_edges) if weighted else None


def path_graph(n: int, weighted: bool = False, seed: int = 0) -> Graph:
    rng = np.random.default_rng(seed)
    src = np.arange(n - 1, dtype=np.int64)
    return from_edges(src, src + 1, _weights(n - 1, weighted, rng), n_vertices=n)


def cycle_graph(n: int, weighted: bool = False, seed: int = 0) -> Graph:
    rng = np.random.default_rng(seed)
    src = np.arange(n, dtype=np.int64)
    return from_edges(src, (src + 1) % n, _weights(n, weighted, rng), n_vertices=n)


def star_graph(n: int, weighted: bool = False, seed: int = 0) -> Graph:
    rng = np.random.default_rng(seed)
    dst = np.arange(1, n, dtype=np.int64)
    return from_edges(np.zeros(n - 1, dtype=np.int64), dst, _weights(n - 1, weighted, rng),
                      n_vertices=n)


def powerlaw_graph(n: int, attach: int = 4, weighted: bool = False, seed: int = 0) -> Graph:
    """Preferential attachment over a repeated-endpoint pool, symmetrised
    (synth.py:44-78): seed ring on `attach` vertices, then each new vertex
    draws `attach` pool indices in one rng.integers call."""
    if n <= attach:
        raise ValueError("need n > attach")
    rng = np.random.default_rng(seed)
    ring = np.arange(attach, dtype=np.int64)
    pool = np.empty(2 * (attach + (n - attach) * attach), dtype=np.int64)
    pool[0:2 * attach:2] = ring
    pool[1:2 * attach:2] = (ring + 1) % attach
    plen = 2 * attach
    src = np.empty(attach + (n - attach) * attach, dtype=np.int64)
    dst = np.empty_like(src)
    src[:attach], dst[:attach] = ring, (ring + 1) % attach
    e = attach
    for v in range(attach, n):
        picks = rng.integers(0, plen, size=attach)
        tg = pool[picks]
        src[e:e + attach] = v
        dst[e:e + attach] = tg
        pool[plen:plen + 2 * attach:2] = v
        pool[plen + 1:plen + 2 * attach:2] = tg
        plen += 2 * attach
        e += attach
    w = _weights(len(src), weighted, rng)
    return from_edges(np.concatenate([src, dst]), np.concatenate([dst, src]),
                      np.concatenate([w, w]) if w is not None else None, n_vertices=n)


GENERATORS = {"path": path_graph, "cycle": cycle_graph, "star": star_graph,
              "powerlaw": powerlaw_graph}


def make_synthetic(spec: str, weighted: bool = False, seed: int = 0) -> Graph:
    name, _, arg = spec.partition(":")
    if name not in GENERATORS:
        raise ValueError(f"unknown synthetic graph {name!r}; choose from {sorted(GENERATORS)}")
    return GENERATORS[name](int(arg) if arg else 1000, weighted=weighted, seed=seed)

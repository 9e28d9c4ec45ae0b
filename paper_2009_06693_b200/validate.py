"""Per-app distribution checks (the CLI's --validate; bench.py:224-364 of the
reference), on the device kernels.

The draws come from the device's `individual_batch` (nd_individual_batch)
over n independent keyed streams on one transit, and PPR walk lengths from a
device `tp_run`; the exact distributions are computed on the host from the
graph's CSR, and the same thresholds as the reference decide pass / FAIL.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .apps import Node2vecParams, make_app, node2vec_factors


@dataclass
class ValidationRow:
    app: str
    check: str
    statistic: float
    threshold: float
    passed: bool

    def line(self) -> str:
        status = "pass" if self.passed else "FAIL"
        return (f"{status}  {self.app:<10} {self.check:<28} "
                f"value={self.statistic:.6f} threshold={self.threshold:g}")


def _host(graph):
    return graph.to_host() if hasattr(graph, "to_host") else graph


def _empirical_counts(values, support):
    idx = np.searchsorted(support, values)
    return np.bincount(idx, minlength=len(support))


def _draw_next_batch(app, graph, transit, n_draws, t_prev=-1, step=0):
    """One app's kernel over n_draws keyed streams (sample ids 0..n-1) on one
    transit (bench.py:245-261)."""
    from .kernels import individual_batch
    g = _host(graph)
    transits = np.full(n_draws, transit, dtype=np.int64)
    t_prev_arr = np.full(n_draws, t_prev, dtype=np.int64)
    sample_ids = np.arange(n_draws, dtype=np.int64)
    zeros = np.zeros(n_draws, dtype=np.int64)
    out = np.empty(n_draws, dtype=np.int64)
    individual_batch(app.kernel_code, app.kernel_params, g.row_offsets, g.col_indices, g.weights,
                     g.per_vertex_weight_prefix, g.per_vertex_max_weight, transits, t_prev_arr,
                     sample_ids, zeros, zeros, 0, step, out)
    return out


def node2vec_exact_distribution(graph, v, t, p, q, convention="reciprocal"):
    """Brute-force normalised pick distribution over v's neighbours (bench.py:264-283)."""
    g = _host(graph)
    f_ret, f_adj, f_far = node2vec_factors(Node2vecParams(p=p, q=q, factor_convention=convention))
    cols, ws = g.neighbors(v)
    mass = {}
    for u, w in zip(cols, ws):
        u = int(u)
        f = f_ret if u == t else (f_adj if g.has_edge(t, u) else f_far)
        mass[u] = mass.get(u, 0.0) + float(w) * f
    total = sum(mass.values())
    return {u: m / total for u, m in mass.items()}


def validate_distributions(app_name, graph, draws=1_000_000, seed=0) -> list:
    """bench.py:286-331: per-app brute-force distribution checks."""
    g = _host(graph)
    rows = []
    if app_name == "deepwalk":
        cols, ws = g.neighbors(0)
        support, inv = np.unique(cols, return_inverse=True)
        exact = np.bincount(inv, weights=ws)
        exact = exact / exact.sum()
        picks = _draw_next_batch(make_app("deepwalk"), g, 0, draws)
        err = float(np.abs(_empirical_counts(picks, support) / draws - exact).max())
        rows.append(ValidationRow("deepwalk", "weighted-pick max |err|", err, 0.005, err < 0.005))
    elif app_name == "node2vec":
        params = {"p": 2.0, "q": 0.5}
        exact = node2vec_exact_distribution(g, 0, 1, **params)
        picks = _draw_next_batch(make_app("node2vec", **params), g, 0, draws, t_prev=1, step=1)
        support = np.asarray(sorted(exact), dtype=np.int64)
        counts = _empirical_counts(picks, support)
        l1 = float(np.abs(counts / draws - np.asarray([exact[int(u)] for u in support])).sum())
        rows.append(ValidationRow("node2vec", "factor-oracle L1", l1, 0.01, l1 < 0.01))
    elif app_name == "khop":
        cols, _ = g.neighbors(0)
        support, inv = np.unique(cols, return_inverse=True)
        expect = np.bincount(inv) / len(cols)
        picks = _draw_next_batch(make_app("khop"), g, 0, draws)
        err = float(np.abs(_empirical_counts(picks, support) / draws - expect).max())
        rows.append(ValidationRow("khop", "uniform-pick max |err|", err, 0.005, err < 0.005))
    elif app_name == "ppr":
        rows.extend(validate_ppr_lengths(graph, n_walks=min(draws, 100_000), seed=seed))
    else:
        rows.append(ValidationRow(app_name, "no distribution oracle", 0.0, 0.0, True))
    return rows


def validate_ppr_lengths(graph, n_walks=100_000, termination=0.01, seed=0) -> list:
    """bench.py:334-364: mean walk length near 1/termination and a geometric
    goodness of fit (chi-square over ~40 buckets up to the 99% quantile)."""
    from scipy import stats as scipy_stats

    from .engine import EngineConfig, make_samples, tp_run
    app = make_app("ppr", termination_probability=termination)
    out = tp_run(app, graph, make_samples(app, graph, n_walks, seed), EngineConfig(seed=seed))
    off, _ = out.final_csr()
    lengths = np.diff(np.asarray(off)) - 1  # sampled vertices per walk (total_sampled)
    mean = float(lengths.mean())
    rows = [ValidationRow("ppr", "mean walk length", mean, 100.0, 97.0 <= mean <= 103.0)]
    p = termination
    max_bucket = int(np.quantile(lengths, 0.99))
    edges = list(range(0, max_bucket, max(1, max_bucket // 40)))
    observed, expected = [], []
    for i, lo in enumerate(edges):
        hi = edges[i + 1] if i + 1 < len(edges) else None
        if hi is None:
            observed.append(int((lengths >= lo).sum()))
            expected.append(n_walks * (1 - p) ** lo)
        else:
            observed.append(int(((lengths >= lo) & (lengths < hi)).sum()))
            expected.append(n_walks * ((1 - p) ** lo - (1 - p) ** hi))
    _, pvalue = scipy_stats.chisquare(observed, expected)
    rows.append(ValidationRow("ppr", "geometric fit p-value", float(pvalue), 0.001, pvalue > 0.001))
    return rows

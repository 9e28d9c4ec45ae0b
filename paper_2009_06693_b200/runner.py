"""Run orchestration (mirror of trawl/bench.py:27-217): RunConfig, RunReport,
run / multi_worker_run / compare_paradigms, all on the device engine.

``paradigm`` is "tp" or "sp" as in the reference (both execute on the GPU;
"gpu" is accepted as an alias of "tp").  Reports carry the same key=value
lines (bench.py:61-84) so existing consumers of the CLI keep working.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

from .apps import make_app
from .core import DEFAULT_STEP_CAP
from .engine import EngineConfig, RunStats, make_samples, sp_run, tp_run
from .errors import OutputMismatchError
from .graph import Graph  # noqa: F401  (type of synthetic graphs)
from .output import LAYOUT_FINAL, SampleSetOutput, render_text
from .sharding import worker_ranges
from .synth import make_synthetic


@dataclass
class RunConfig:
    app: str = "deepwalk"
    app_params: dict = field(default_factory=dict)
    paradigm: str = "tp"
    graph_path: Optional[str] = None
    synth: Optional[str] = None
    weighted: bool = False
    undirected: bool = False
    seed: int = 0
    num_samples: int = 1000
    workers: int = 1
    layout: str = LAYOUT_FINAL
    output_path: Optional[str] = None
    report_path: Optional[str] = None
    step_cap: int = DEFAULT_STEP_CAP
    use_kernels: bool = True

    def load_graph(self):
        """bench.py:45-50: file graphs keyed on the run seed; synthetic graphs
        built with the run seed.  Edge-list files are parsed and built on the
        device (DeviceGraph.from_edge_list: same graph, ids, remap and errors as
        the reference's load_edge_list)."""
        if self.graph_path:
            from .graph import DeviceGraph
            return DeviceGraph.from_edge_list(self.graph_path, weighted=self.weighted,
                                              undirected=self.undirected, seed=self.seed)
        return make_synthetic(self.synth or "powerlaw:1000", weighted=self.weighted, seed=self.seed)


@dataclass
class RunReport:
    config: RunConfig
    stats: RunStats
    wall_s: float

    def lines(self) -> list[str]:
        s = self.stats
        small, medium, large = s.group_totals()
        out = [
            f"app={self.config.app}",
            f"paradigm={s.paradigm}",
            f"samples={s.n_samples}",
            f"seed={self.config.seed}",
            f"workers={self.config.workers}",
            f"steps={s.n_steps}",
            f"total_s={s.total_s:.6f}",
            f"build_s={s.build_s:.6f}",
            f"sample_s={s.sample_s:.6f}",
            f"build_share={s.build_s / s.total_s if s.total_s > 0 else 0.0:.4f}",
            f"throughput_samples_per_s={s.throughput():.2f}",
            f"adjacency_fetches={s.adjacency_fetches}",
            f"groups.small={small}",
            f"groups.medium={medium}",
            f"groups.large={large}",
        ]
        for t in s.timings:
            out.append(f"step.{t.step}.build_s={t.build_s:.6f}")
            out.append(f"step.{t.step}.sample_s={t.sample_s:.6f}")
        return out

    def write(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("\n".join(self.lines()) + "\n")


def _engine_for(paradigm: str):
    if paradigm == "sp":
        return sp_run
    if paradigm in ("tp", "gpu"):
        return tp_run
    raise ValueError(f"unknown paradigm {paradigm!r}")


def _engine_config(config: RunConfig) -> EngineConfig:
    return EngineConfig(seed=config.seed, n_workers=1, step_cap=config.step_cap,
                        use_kernels=config.use_kernels)


def run_single(config: RunConfig, graph) -> SampleSetOutput:
    app = make_app(config.app, **config.app_params)
    samples = make_samples(app, graph, config.num_samples, config.seed)
    return _engine_for(config.paradigm)(app, graph, samples, _engine_config(config))


def split_ranges(n: int, workers: int):
    return worker_ranges(n, workers)


def multi_worker_run(config: RunConfig, graph) -> SampleSetOutput:
    """Contiguous per-worker sample ranges with global ids (bench.py:123-153);
    each range is one device run, outputs concatenated in id order."""
    if config.workers <= 1:
        return run_single(config, graph)
    import numpy as np
    engine = _engine_for(config.paradigm)
    outs = []
    for lo, hi in split_ranges(config.num_samples, config.workers):
        app = make_app(config.app, **config.app_params)
        outs.append(engine(app, graph, make_samples(app, graph, hi - lo, config.seed, lo=lo),
                           _engine_config(config)))
    stats = RunStats(paradigm=config.paradigm, n_samples=config.num_samples)
    for o in outs:
        stats.timings.extend(o.stats.timings)
        stats.adjacency_fetches += o.stats.adjacency_fetches
        stats.total_s += o.stats.total_s
    return _concat(outs, graph, stats)


def _concat(outs, graph, stats) -> SampleSetOutput:
    import numpy as np

    def cat(parts):
        return np.concatenate(parts) if parts else np.empty(0, dtype=np.int64)

    n_steps = max((o.n_steps for o in outs), default=0)
    ids = cat([o.sample_ids for o in outs])
    roots = cat([o.roots for o in outs])
    roots_off = np.concatenate([[0], np.cumsum(cat([np.diff(o.roots_off) for o in outs]))])
    foff_parts, fids = [], []
    base = 0
    for o in outs:
        off, fi = o.final_csr()
        foff_parts.append(off[1:] + base)
        fids.append(fi)
        base += len(fi)
    final_off = np.concatenate([[0]] + foff_parts)
    kw = {}
    if outs and outs[0].chain_vals is not None:
        clen = cat([np.diff(o.chain_off) for o in outs])
        kw = dict(chain_off=np.concatenate([[0], np.cumsum(clen)]),
                  chain_vals=cat([o.chain_vals for o in outs]))
    else:
        S = n_steps
        cnt = np.concatenate([np.pad(o.step_counts, ((0, S - o.step_counts.shape[0]), (0, 0)))
                              for o in outs], axis=1) if outs else np.zeros((0, 0), np.int64)
        vals = []
        for st in range(S):
            for o in outs:
                if st < o.step_counts.shape[0]:
                    b = o._step_base()
                    vals.append(o.step_vals[b[st]:b[st + 1]])
        kw = dict(step_counts=cnt, step_vals=cat(vals))
        if outs and any(o.rec_counts is not None and o.rec_t is not None for o in outs):
            # recorded edges, step-major like step_vals (multi_worker_run keeps them)
            rc, rt, rv = [], [], []
            for o in outs:
                c = o.rec_counts if o.rec_counts is not None else np.zeros((0, o.n_samples),
                                                                             np.int64)
                rc.append(np.pad(np.asarray(c, np.int64), ((0, S - c.shape[0]), (0, 0))))
            for st in range(S):
                for o in outs:
                    if o.rec_counts is None or o.rec_t is None or st >= len(o.rec_counts):
                        continue
                    tot = np.asarray(o.rec_counts).sum(axis=1)
                    a = int(tot[:st].sum())
                    b = a + int(tot[st])
                    rt.append(o.rec_t[a:b])
                    rv.append(o.rec_v[a:b])
            kw.update(rec_counts=np.concatenate(rc, axis=1), rec_t=cat(rt), rec_v=cat(rv))
    return SampleSetOutput(ids, roots_off, roots, n_steps, remap=getattr(graph, "remap", None),
                           stats=stats, final_off=final_off, final_ids=cat(fids), **kw)


def run(config: RunConfig, graph=None):
    """Load (or take) a graph, run, build the report; loading is untimed."""
    if graph is None:
        graph = config.load_graph()
    t0 = time.perf_counter()
    output = multi_worker_run(config, graph)
    wall = time.perf_counter() - t0
    return output, RunReport(config=config, stats=output.stats, wall_s=wall)


@dataclass
class ComparisonReport:
    sp_report: RunReport
    tp_report: RunReport
    outputs_equal: bool

    @property
    def throughput_ratio_tp_over_sp(self) -> float:
        return self.tp_report.stats.throughput() / self.sp_report.stats.throughput()

    @property
    def fetch_ratio_sp_over_tp(self) -> float:
        tp = self.tp_report.stats.adjacency_fetches
        return self.sp_report.stats.adjacency_fetches / tp if tp else float("inf")

    def lines(self) -> list[str]:
        tp = self.tp_report.stats
        return [
            f"outputs_equal={self.outputs_equal}",
            f"throughput_sp={self.sp_report.stats.throughput():.2f}",
            f"throughput_tp={tp.throughput():.2f}",
            f"throughput_ratio_tp_over_sp={self.throughput_ratio_tp_over_sp:.4f}",
            f"fetches_sp={self.sp_report.stats.adjacency_fetches}",
            f"fetches_tp={tp.adjacency_fetches}",
            f"fetch_ratio_sp_over_tp={self.fetch_ratio_sp_over_tp:.4f}",
            f"tp_build_index_share={tp.build_s / tp.total_s if tp.total_s > 0 else 0.0:.4f}",
        ]


def compare_paradigms(config: RunConfig, graph=None) -> ComparisonReport:
    """Both paradigms on one config; outputs must match byte for byte."""
    if graph is None:
        graph = config.load_graph()
    reports, texts = {}, {}
    for paradigm in ("sp", "tp"):
        cfg = RunConfig(**{**config.__dict__, "paradigm": paradigm})
        output, report = run(cfg, graph)
        reports[paradigm] = report
        texts[paradigm] = render_text(output, config.layout)
    if texts["sp"] != texts["tp"]:
        raise OutputMismatchError(f"sp and tp outputs differ for app={config.app} seed={config.seed}")
    return ComparisonReport(reports["sp"], reports["tp"], True)

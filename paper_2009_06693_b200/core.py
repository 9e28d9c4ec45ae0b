"""The sampling-application API (mirror of trawl/core.py:27-203).

``SamplingApp`` keeps the reference's field names and meanings
(steps / sample_size / next / individual-vs-collective sampling_type /
unique / transit_source / needs_prev2 / records_edges / chain_walk /
kernel_code / params) so an app built with ``make_app`` — ours or the
reference's — is accepted unchanged by ``tp_run``.  The device engine
does not call ``next_fn`` per slot: it recognises the app by
``kernel_code`` (individual apps, trawl/kernels/_pykernels.py:32-36) or by
``name`` + ``params`` (collective apps, trawl/apps.py:247-386) and runs
the matching CUDA kernel with the same draw protocol.  An app that only
carries a custom Python ``next_fn`` is rejected with
``UnsupportedAppError`` — there is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

NULL_VERTEX = -1                 # core.py:27
INF_STEPS = math.inf             # core.py:28
INDIVIDUAL = "individual"        # core.py:30
COLLECTIVE = "collective"        # core.py:31
TRANSITS_PREV_STEP = "prev_step"  # core.py:34
TRANSITS_ROOT_PICK = "root_pick"  # core.py:35
DEFAULT_STEP_CAP = 10_000        # core.py:37

_EMPTY = np.empty(0, dtype=np.int64)


@dataclass
class SamplingApp:
    """One application: same fields as trawl.core.SamplingApp (core.py:134-165)."""

    name: str
    sampling_type: str
    steps: float
    sample_size: Callable[[int], int]
    next_fn: Callable
    unique: Callable[[int], bool] = lambda step: False
    transit_source: str = TRANSITS_PREV_STEP
    step_transits_fn: Optional[Callable] = None
    init_roots: Optional[Callable] = None
    post_step: Optional[Callable] = None
    needs_prev2: bool = False
    records_edges: bool = False
    chain_walk: bool = False
    kernel_code: Optional[int] = None
    select_batch: Optional[Callable] = None
    kernel_params: np.ndarray = field(default_factory=lambda: np.zeros(0))
    params: dict = field(default_factory=dict)

    def is_individual(self) -> bool:
        return self.sampling_type == INDIVIDUAL


class Sample:
    """Host view of one sample (core.py:42-131): ``id``, ``roots``, per-step
    slot arrays and recorded edges.  Device runs produce these lazily from
    the compacted device output (``SampleSetOutput.samples``)."""

    __slots__ = ("id", "roots", "step_vertices", "recorded_edges", "graph", "step")

    def __init__(self, sample_id: int, roots, graph=None):
        self.id = int(sample_id)
        self.roots = np.asarray(roots, dtype=np.int64)
        self.step_vertices: list[np.ndarray] = []
        self.recorded_edges: list[tuple[np.ndarray, np.ndarray]] = []
        self.graph = graph
        self.step = 0

    def n_steps_run(self) -> int:
        return len(self.step_vertices)

    def vertices_at(self, step: int) -> np.ndarray:
        """Non-NULL vertices of a step; roots for step -1 (core.py:84-97)."""
        if step == -1:
            return self.roots
        if step >= len(self.step_vertices):
            return _EMPTY
        sv = self.step_vertices[step]
        return sv[sv != NULL_VERTEX]

    def total_sampled(self) -> int:
        return int(sum(int((sv != NULL_VERTEX).sum()) for sv in self.step_vertices))

    def size(self) -> int:
        return len(self.roots) + self.total_sampled()

    def final_vertices(self) -> np.ndarray:
        parts = [self.roots] + [self.vertices_at(i) for i in range(len(self.step_vertices))]
        return np.concatenate(parts)

    def prev_vertex(self, back: int, pos: int) -> int:
        return int(self.vertices_at(self.step - back)[pos])


def transit_count_hint(app, n_roots: int) -> int:
    """Transits at step 0 (core.py:187-192): 1 for root-pick apps, else the
    root count."""
    if getattr(app, "transit_source", TRANSITS_PREV_STEP) == TRANSITS_ROOT_PICK:
        return 1 if n_roots else 0
    return n_roots

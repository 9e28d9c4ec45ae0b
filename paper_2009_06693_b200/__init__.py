"""NextDoor on B200: transit-parallel graph sampling (arXiv 2009.06693).

Host API mirrors the reference ``trawl`` package (make_app, SamplingApp,
EngineConfig, tp_run/sp_run, SampleSetOutput, render_text); every run
executes in hand-written sm_100a CUDA kernels behind the C-ABI in
include/nextdoor_b200.h.  There is no CPU fallback: the engine raises if
the CUDA library is missing.
"""

from .apps import APP_NAMES, make_app
from .core import (COLLECTIVE, INDIVIDUAL, INF_STEPS, NULL_VERTEX, Sample,
                   SamplingApp)
from .errors import (ContractViolationError, DeviceError, SamplerStallError,
                     TrawlError, UnsupportedAppError)
from .output import (LAYOUT_FINAL, LAYOUT_PER_STEP, SampleSetOutput, emit,
                     render_text)
from .engine import (DeviceRun, EngineConfig, RunStats, StepTiming, make_samples,
                     run_device, sp_run, tp_run)
from .graph import DeviceGraph, Graph, from_edges, load_cache, load_edge_list, save_cache
from .rng import RngStream, key_u64, key_uniform
from .sharding import worker_ranges

__version__ = "0.1.0"
BACKEND_NAME = "cuda-sm100a"

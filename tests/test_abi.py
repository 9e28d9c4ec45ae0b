"""The C-ABI library loads on a CPU box and exports every entry point that
include/nextdoor_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

from paper_2009_06693_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                   "nextdoor_b200.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("nd_individual_batch", "nd_segmented_prefix_sum", "nd_segment_max",
                 "nd_run_walk", "nd_run_individual", "nd_run_collective", "nd_transit_schedule",
                 "nd_graph_create", "nd_graph_rmat", "nd_result_copy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert set(_lib.SIGNATURES) == set(declared())
    L = _lib.load()
    assert L.nd_version() == 1


def test_integration_guide_covers_every_entry_point():
    """INTEGRATION.md maps every declared entry point to the reference
    interface it replaces (or says it has none)."""
    doc = open(os.path.join(os.path.dirname(HDR), "..", "INTEGRATION.md")).read()
    missing = [n for n in declared() if n not in doc]
    assert not missing, missing


def test_engine_fails_loudly_without_cuda():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2009_06693_b200 import make_app, DeviceError
    from paper_2009_06693_b200.engine import run_device
    with pytest.raises(DeviceError):
        run_device(make_app("deepwalk"), None, n_samples=1)


def test_concurrency_share_is_thread_local_setting():
    """nd_set_concurrency: k >= 1 accepted, k < 1 rejected; no GPU needed."""
    L = _lib.load()
    assert L.nd_set_concurrency(2) == 0
    assert L.nd_set_concurrency(0) != 0
    assert L.nd_set_concurrency(1) == 0


def test_gpu_share_nests_and_restores():
    from paper_2009_06693_b200.engine import gpu_share
    with gpu_share(3) as a:
        assert gpu_share._state().k == 3
        with gpu_share(2):
            assert gpu_share._state().k == 2
        assert gpu_share._state().k == 3
    assert gpu_share._state().k == 1 and a.k == 3

"""Host-side mirror of the reference API (CPU): the cases the reference's own
tests pin for these helpers.

* Graph.weighted_pick thresholds on prefix [1, 4] (tests/test_graph.py:65-73):
  r = 0.10 -> 1, 0.2499 -> 1, 0.25 -> 2, 0.90 -> 2; NoNeighborsError on an
  empty row (graph.py:90-91); has_edge on the sorted row.
* partition_work_classes thresholds 31/32/1024/1025 and the dense per-class
  scheduling index; subgroup_size = max(1, 32 // m)
  (tests/test_transit_schedule.py).
* dedup / fallback boundary (output.py:27-40, tests/test_postprocess.py).
"""

import numpy as np
import pytest


def test_weighted_pick_thresholds_and_has_edge():
    from paper_2009_06693_b200.errors import NoNeighborsError
    from paper_2009_06693_b200.graph import from_edges
    # vertex 0 -> 1 (w 1), 0 -> 2 (w 3): prefix [1, 4]; vertex 3 has no edges
    g = from_edges([0, 0, 1, 2], [1, 2, 2, 0], [1.0, 3.0, 1.0, 1.0], n_vertices=4)
    # the prefix is a device computation (nd_segmented_prefix_sum); on CPU set
    # the sequential per-row prefix it produces
    g._prefix = np.concatenate([np.cumsum(g.weights[g.row_offsets[v]:g.row_offsets[v + 1]])
                                for v in range(g.n_vertices)])
    assert g._prefix.tolist() == [1.0, 4.0, 1.0, 1.0]
    for r, exp in ((0.10, 1), (0.2499, 1), (0.25, 2), (0.90, 2)):
        assert g.weighted_pick(0, r) == exp, r
    with pytest.raises(NoNeighborsError):
        g.weighted_pick(3, 0.5)
    assert g.has_edge(0, 2) and g.has_edge(1, 2) and not g.has_edge(1, 0) and not g.has_edge(3, 0)


def test_work_classes_and_subgroups():
    from paper_2009_06693_b200.schedule import TransitGroup, partition_work_classes, subgroup_size
    sizes = {10: 31, 11: 32, 12: 1024, 13: 1025, 14: 1, 15: 500}
    groups = [TransitGroup(t, np.arange(n)) for t, n in sizes.items()]
    sched = partition_work_classes(groups, 1)
    assert [g.transit for g in sched.small] == [10, 14]
    assert [g.transit for g in sched.medium] == [11, 12, 15]
    assert [g.transit for g in sched.large] == [13]
    assert sched.class_counts() == (2, 3, 1) and len(sched.all_groups()) == 6
    assert [sched.scheduling_index[t] for t in (10, 14, 11, 12, 15, 13)] == [0, 1, 0, 1, 2, 0]
    # work = members * m: 8 members x m=4 = 32 is medium
    assert partition_work_classes([TransitGroup(1, np.arange(8))], 4).class_counts() == (0, 1, 0)
    assert [subgroup_size(m) for m in (1, 2, 25, 32, 33, 250)] == [32, 16, 1, 1, 1, 1]


def test_dedup_and_fallback_boundary():
    from paper_2009_06693_b200.output import dedup_rows, fallback_check
    assert dedup_rows(np.array([5, -1, 3, 5, 3, -1, 9])).tolist() == [3, 5, 9]
    assert dedup_rows(np.array([-1, -1])).tolist() == []
    # SP fallback iff 0 < distinct < m_i
    assert not fallback_check(0, 4) and fallback_check(1, 4) and fallback_check(3, 4)
    assert not fallback_check(4, 4) and not fallback_check(5, 4)


def test_validation_row_format_and_cli_flag():
    """validate.ValidationRow prints the reference's line (bench.py:224-236)
    and the CLI accepts --validate (cli.py:58)."""
    from paper_2009_06693_b200.cli import build_parser
    from paper_2009_06693_b200.validate import ValidationRow, _empirical_counts
    import numpy as np
    row = ValidationRow("deepwalk", "weighted-pick max |err|", 0.0012345, 0.005, True)
    assert row.line() == ("pass  deepwalk   weighted-pick max |err|      value=0.001234 "
                          "threshold=0.005")
    assert ValidationRow("ppr", "geometric fit p-value", 0.0, 0.001, False).line().startswith("FAIL  ppr")
    assert np.array_equal(_empirical_counts(np.array([3, 1, 3, 7]), np.array([1, 3, 7])), [1, 2, 1])
    args = build_parser().parse_args(["--app", "khop", "--synth", "cycle:8", "--validate"])
    assert args.validate is True

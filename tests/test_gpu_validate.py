"""The distribution checks of the CLI's --validate (bench.py:224-364 of the
reference) on the device kernels, with the reference's own test cases:
tests/test_bench.py:68-74, tests/test_acceptance.py:119-156 and
tests/test_cli.py:89-92."""

import pytest

pytestmark = pytest.mark.gpu


def test_validation_rows_pass():
    from paper_2009_06693_b200.graph import from_edges
    from paper_2009_06693_b200.validate import validate_distributions
    two = from_edges([0, 0], [1, 2], [1.0, 3.0], n_vertices=3)
    five = from_edges([0, 0, 0, 0, 1, 1, 2], [1, 2, 3, 4, 0, 2, 3],
                      [1.5, 2.0, 0.5, 3.0, 1.0, 1.0, 1.0], n_vertices=5)
    for app, g in (("deepwalk", two), ("node2vec", five), ("khop", five)):
        rows = validate_distributions(app, g, draws=1_000_000)
        assert rows and all(r.passed for r in rows), [r.line() for r in rows]
    assert validate_distributions("deepwalk", two, draws=1_000_000)[0].statistic < 0.005


def test_ppr_length_law():
    from paper_2009_06693_b200.synth import cycle_graph
    from paper_2009_06693_b200.validate import validate_ppr_lengths
    mean_row, fit_row = validate_ppr_lengths(cycle_graph(1000, weighted=True, seed=2),
                                             n_walks=100_000, termination=0.01, seed=0)
    assert 97.0 <= mean_row.statistic <= 103.0
    assert fit_row.statistic > 0.001


def test_cli_validate_flag(capsys):
    from paper_2009_06693_b200.cli import main
    assert main(["--app", "khop", "--synth", "cycle:8", "--validate"]) == 0
    assert "pass" in capsys.readouterr().out

"""cli_harness: config round-trip, CSV/table emit and parse,
exit codes for config errors (CPU), and the convergence runs on the GPU
(SPEC.md acceptance 2, 3, 5, 6: PAPER.md Tables 1-3 rows)."""
import numpy as np
import pytest

from paper_2504_07269_b200 import cli


def test_config_roundtrip_idempotent():
    text = "spatial=square:16\ntemporal=graded:1.5\nT=2.5\nnt=8  # comment\nlevels=1\nsolver=bs\n"
    c = cli.RunConfig.parse(text)
    assert c.spatial == "square:16" and c.temporal == "graded:1.5" and c.T == 2.5 and c.nt == 8
    s1 = c.serialize()
    assert cli.RunConfig.parse(s1).serialize() == s1


@pytest.mark.parametrize("bad", ["spatial=circle:3", "temporal=graded:0.5", "T=-1", "solver=lu",
                                 "nosuchkey=1", "nt=abc", "problem=foo"])
def test_config_errors(bad):
    with pytest.raises(cli.ConfigError):
        cli.RunConfig.parse(bad)


def test_emit_csv_roundtrip_and_table():
    rows = [cli.ConvergenceRow(61504, 0.0442, 0.078125, 3.19e-3, None, 2.397e-1, None, 0.11, 229.3),
            cli.ConvergenceRow(508032, 0.0221, 0.0390625, 8.143e-4, 1.97, 1.2003e-1, 0.998, 0.31, 700.7)]
    text = cli.emit(rows, "csv")
    lines = text.strip().splitlines()
    assert lines[0] == cli.HEADER and lines[1].split(",")[4] == "-" and len(lines) == 3
    back = cli.parse_csv(text)
    for a, b in zip(rows, back):
        assert a.n == b.n
        for k in ("hx", "ht", "errL2", "errH1", "solve_s", "kappa2"):
            assert abs(getattr(a, k) - getattr(b, k)) <= 5e-4 * abs(getattr(a, k))
    assert back[0].eocL2 is None and abs(back[1].eocL2 - 1.97) < 1e-3
    tab = cli.emit(rows, "table")
    assert "kappa2" in tab and tab.count("\n") == 3
    assert cli.emit(rows[:1], "csv").count("\n") == 2          # header + one data line


def test_cli_exit_code_config_error(capsys):
    assert cli.main(["convergence", "--spatial", "hexagon:4"]) == 3
    assert cli.main(["solve", "--solver", "qr"]) == 3
    # memory guard: level 4 of the paper preset needs far more than 0.01 GiB
    assert cli.main(["convergence", "--levels", "4", "--mem-guard-gib", "0.01"]) == 3


@pytest.mark.gpu
def test_paper_table2_rows_fd():
    """SPEC.md:508 / acceptance 2: paper preset, J_max = 1, FD -> n in {61504, 508032},
    L2 ~ {3.2e-3, 8.1e-4} (15%), H1 ~ {2.4e-1, 1.2e-1}, kappa2 ~ {2.3e2, 7.0e2} (5%)."""
    rows = cli.run_convergence(cli.RunConfig(levels=1))
    assert [r.n for r in rows] == [61504, 508032]
    for r, l2, h1, k in zip(rows, (3.2e-3, 8.1e-4), (2.4e-1, 1.2e-1), (2.3e2, 7.0e2)):
        assert abs(r.errL2 - l2) / l2 < 0.15 and abs(r.errH1 - h1) / h1 < 0.15
        assert abs(r.kappa2 - k) / k < 0.05
    assert 1.8 <= rows[1].eocL2 <= 2.2 and 0.9 <= rows[1].eocH1 <= 1.1


@pytest.mark.gpu
def test_convergence_orders_and_variant_agreement():
    """Acceptance 3 and 6: levels 0-2 eoc bands; BS and FD errors agree to 3 s.f."""
    fd = cli.run_convergence(cli.RunConfig(levels=2))
    bs = cli.run_convergence(cli.RunConfig(levels=2, solver="bs"))
    for r in fd[1:]:
        assert 1.8 <= r.eocL2 <= 2.2 and 0.9 <= r.eocH1 <= 1.1
    for a, b in zip(fd, bs):
        assert abs(a.errL2 - b.errL2) / a.errL2 < 5e-4 and abs(a.errH1 - b.errH1) / a.errH1 < 5e-4
        assert b.kappa2 == 1.0


@pytest.mark.gpu
def test_graded_table3_row1(tmp_path):
    """Acceptance 5: graded q = 1.5, n_t = 64 -> h_t within 2% of 1.167e-1, kappa2 = 1.1e2
    (5%), L2 = 3.2e-3 (15%), FD succeeds; written through the CLI as CSV."""
    out = tmp_path / "t3.csv"
    assert cli.main(["solve", "--temporal", "graded:1.5", "--format", "csv", "--out", str(out)]) == 0
    (r,) = cli.parse_csv(out.read_text())
    assert abs(r.ht - 1.167e-1) / 1.167e-1 < 0.02
    assert abs(r.kappa2 - 1.1e2) / 1.1e2 < 0.05 and abs(r.errL2 - 3.2e-3) / 3.2e-3 < 0.15


@pytest.mark.gpu
def test_zero_problem_row():
    """zero-source preset with psi0 = 0 -> zero solution, errors 0."""
    (r,) = cli.run_convergence(cli.RunConfig(spatial="square:8", nt=4, T=1.0, problem="zero"))
    assert r.errL2 == 0.0 and r.errH1 == 0.0

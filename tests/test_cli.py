"""CLI front end and run artefacts, host side: config
parsing and validation, and the artefact formats.  The GPU runs are in
tests/test_gpu_cli.py."""

import numpy as np
import pytest

from paper_2209_10886_b200 import artifacts, cli
from paper_2209_10886_b200.discretization import ProblemSpec
from paper_2209_10886_b200.driver import SolveReport
from paper_2209_10886_b200.indexing import Partition


def test_defaults_and_flags_override_file(tmp_path):
    f = tmp_path / "run.cfg"
    f.write_text("# a comment\nn1 = 5\nn2 = 3   # trailing comment\nprecond = sp\nbsp-seam = literal\ntol=1e-9\n")
    cfg = cli.resolve(["--config", str(f), "--n2", "4", "--mono-check", "--mono-field", "m.npy"])
    assert (cfg["n1"], cfg["n2"], cfg["precond"], cfg["bsp_seam"], cfg["tol"]) == (5, 4, "sp", "literal", 1e-9)
    assert cfg["mono_check"] is True and cfg["maxit"] == 200
    assert cfg["scatterer_obj"].radius == 1.0


@pytest.mark.parametrize("argv,key", [
    (["--n1", "0"], "n1"), (["--cells", "3"], "cells"), (["--precond", "ilu"], "precond"),
    (["--bsp-seam", "x"], "bsp_seam"), (["--tol", "-1"], "tol"), (["--kappa", "abc"], "kappa"),
    (["--scatterer", "1,2"], "scatterer"), (["--workers", "0"], "workers"), (["--blocks", "0"], "blocks"),
    (["--mono-check"], "mono_check"), (["--table", "5by5"], "table"), (["--config", "/nonexistent"], "config"),
])
def test_config_errors_name_the_key(argv, key):
    with pytest.raises(cli.ConfigError) as ei:
        cli.resolve(argv)
    assert ei.value.key == key


def test_config_file_errors(tmp_path):
    f = tmp_path / "bad.cfg"
    f.write_text("n1 = 2\ncolour = red\n")
    with pytest.raises(cli.ConfigError, match="colour"):
        cli.resolve(["--config", str(f)])
    f.write_text("n1 2\n")
    with pytest.raises(cli.ConfigError, match="line 1"):
        cli.resolve(["--config", str(f)])


def test_main_exit_1_on_config_error(capsys):
    assert cli.main(["--precond", "ilu"]) == 1
    assert "precond" in capsys.readouterr().err


def test_scatterer_none_and_table_parse():
    cfg = cli.resolve(["--scatterer", "none", "--table", "5x5,5x10"])
    assert cfg["scatterer_obj"] is None and cfg["table_parts"] == [(5, 5), (5, 10)]


def test_schedule_format_matches_oracle():
    from oracle.sweeps import format_trace
    recs = [(1, "forward", [(1, 1)]), (2, "forward", [(2, 1), (1, 2)]), (3, "residual", [(1, 1), (2, 1)])]
    assert artifacts.format_schedule(recs) == format_trace(recs)
    assert artifacts.format_schedule(recs).splitlines()[1] == "step=2 phase=forward solves=(2,1);(1,2)"


def test_residuals_and_report_formats():
    rep = SolveReport(iterations=2, steps_per_iteration=4, total_sequential_steps=8,
                      residual_history=[1.0, 0.1, 1e-7], wall_time=0.5, converged=True)
    text = artifacts.format_residuals(rep.residual_history)
    assert text.splitlines() == ["iteration,relative_residual", "0,1", "1,0.10000000000000001", "2,9.9999999999999995e-08"]
    spec = ProblemSpec(kappa=6.0, cells_per_side=8)
    r = artifacts.format_report(rep, spec, Partition(2, 3), "bsp")
    assert "iterations = 2" in r and "steps_per_iteration = 4" in r and "wall_time" not in r
    assert "wall_time = 0.500000" in artifacts.format_report(rep, spec, Partition(2, 3), "bsp", timings=True)


def test_field_format_coordinates():
    spec = ProblemSpec(kappa=6.0, cells_per_side=4, subdomain_side=1.0)
    part = Partition(2, 3)
    field = (np.arange(12 * 8) + 1j * np.arange(12 * 8)[::-1]).reshape(12, 8)
    lines = artifacts.format_field(spec, part, field).splitlines()
    assert lines[0] == "# kappa=6 N1=2 N2=3 n=4"
    assert len(lines) == 1 + 96
    h = 0.25
    x, y, re, im = (float(v) for v in lines[1 + 5 * 8 + 6].split(","))  # global row 5, column 6
    assert (x, y) == pytest.approx((-0.5 + (6 + 0.5) * h, -0.5 + (5 + 0.5) * h))
    assert (re, im) == (field[5, 6].real, field[5, 6].imag)
    with pytest.raises(ValueError):
        artifacts.format_field(spec, part, field[:, :4])


def test_table_rows():
    rep = SolveReport(iterations=7, steps_per_iteration=16, total_sequential_steps=112,
                      residual_history=[1.0], wall_time=0.25, converged=True)
    assert artifacts.table_row(5, 5, "sp", rep) == "5,5,sp,7,16,0.250000,true,\n"
    assert artifacts.table_row(5, 10, "bsp", error="boom, bad") == "5,10,bsp,,,,false,boom; bad\n"

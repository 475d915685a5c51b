"""GPU: the SPEC front end end to end (SPEC.md:492-505 examples) -- artefact
files, exit codes, byte-identical reruns and the Table-1 sweep."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200 import cli  # noqa: E402


def _read(d, name):
    return (d / name).read_text()


def test_sp_5x5_reports_ns16(tmp_path):
    out = tmp_path / "a"
    assert cli.main(["--n1", "5", "--n2", "5", "--precond", "sp", "--out", str(out)]) == 0
    rep = _read(out, "report.txt")
    assert "steps_per_iteration = 16" in rep and "converged = true" in rep
    it = int(rep.split("iterations = ")[1].split()[0])
    assert len(_read(out, "residuals.csv").splitlines()) == 1 + it + 1  # header + iterations 0..it
    sched = _read(out, "schedule.txt").splitlines()
    assert len(sched) == 16 and sched[0].startswith("step=1 phase=forward solves=")
    field = _read(out, "field.csv").splitlines()
    assert field[0].startswith("# kappa=") and len(field) == 1 + 25 * 20 * 20


def test_1x1_zero_iterations(tmp_path):
    out = tmp_path / "b"
    assert cli.main(["--n1", "1", "--n2", "1", "--out", str(out)]) == 0
    assert "iterations = 0" in _read(out, "report.txt")
    assert len(_read(out, "field.csv").splitlines()) == 1 + 400


def test_seam_modes_differ_from_iteration_1(tmp_path):
    a, b = tmp_path / "dedup", tmp_path / "literal"
    base = ["--n1", "3", "--n2", "3", "--precond", "bsp", "--blocks", "2"]
    assert cli.main(base + ["--bsp-seam", "dedup", "--out", str(a)]) == 0
    assert cli.main(base + ["--bsp-seam", "literal", "--out", str(b)]) == 0
    ra, rb = _read(a, "residuals.csv").splitlines(), _read(b, "residuals.csv").splitlines()
    assert ra[:2] == rb[:2]           # header + iteration 0 (= 1)
    assert ra[2] != rb[2]             # iteration 1 onward differs


def test_rerun_byte_identical(tmp_path):
    """SPEC acceptance 8: report, residuals and field byte-identical for
    workers in {1, 2, 4} on a 3x3 run."""
    base = ["--n1", "3", "--n2", "3", "--precond", "bsp"]
    outs = []
    for w in (1, 2, 4):
        d = tmp_path / f"w{w}"
        assert cli.main(base + ["--out", str(d), "--workers", str(w)]) == 0
        outs.append(d)
    for name in ("residuals.csv", "schedule.txt", "field.csv", "report.txt"):
        assert _read(outs[0], name) == _read(outs[1], name) == _read(outs[2], name), name


def test_not_converged_exit_2(tmp_path):
    assert cli.main(["--n1", "4", "--n2", "4", "--precond", "none", "--maxit", "2",
                     "--tol", "1e-12", "--out", str(tmp_path / "c")]) == 2
    assert "converged = false" in _read(tmp_path / "c", "report.txt")


def test_experiment_table(tmp_path):
    out = tmp_path / "t"
    assert cli.main(["--table", "5x5,5x10,1x1", "--out", str(out)]) == 0
    rows = _read(out, "table.csv").splitlines()
    assert rows[0] == "N1,N2,precond,ni,ns,t,converged,error"
    assert len(rows) == 1 + 6
    ns = [r.split(",")[4] for r in rows[1:5]]
    assert ns == ["16", "10", "26", "10"]  # SPEC.md:503 (Table 1 ns columns)
    ni = {(r.split(",")[0], r.split(",")[1], r.split(",")[2]): int(r.split(",")[3]) for r in rows[1:5]}
    assert ni[("5", "5", "bsp")] >= ni[("5", "5", "sp")]

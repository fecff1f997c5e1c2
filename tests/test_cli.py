"""The `paco` command-line harness."""

import io
import subprocess
import sys

import pytest

from paper_2011_01441_b200 import cli


def test_header_is_the_spec_schema():
    assert cli.HEADER.split(",")[:16] == (
        "algo,n,m,k,p,Z,L,seed,mode,time_s,work_total,work_max,miss_total,miss_max,temp_peak,ok").split(",")


def test_spec_rejections(tmp_path):
    with pytest.raises(ValueError, match="outside this build"):
        cli.run_spec({"algo": "lcs"}, io.StringIO())
    with pytest.raises(ValueError, match="repeats >= 3"):
        cli.run_spec({"algo": "mm", "mode": "parallel", "repeats": "1"}, io.StringIO())
    spec = tmp_path / "s.txt"
    spec.write_text("algo = mm   # comment\nn = 64,128\np=1,3\n")
    assert cli.read_spec(str(spec)) == {"algo": "mm", "n": "64,128", "p": "1,3"}


def test_bad_arguments_exit_2():
    r = subprocess.run([sys.executable, "-m", "paper_2011_01441_b200.cli", "mm", "--n", "8", "--p", "3",
                        "--variant", "hetero", "--weights", "1,2"], capture_output=True, text=True)
    assert r.returncode == 2 and "weights" in r.stderr


@pytest.mark.gpu
def test_mm_and_strassen_rows_pass():
    for semiring in ("int", "minplus-sat", "maxplus", "f32", "bf16", "minplus", "f64"):
        for variant in ("paco", "one-piece"):
            row, ok = cli.run_mm(200, 150, 300, 3, variant=variant, semiring=semiring, mode="parallel")
            f = dict(zip(cli.HEADER.split(","), row.split(",")))
            assert ok and f["ok"] == "pass" and float(f["time_s"]) > 0, (semiring, variant, row)
            assert int(f["work_total"]) >= 200 * 150 * 300
    row, ok = cli.run_mm(300, 200, 100, 2, variant="hetero", weights=[1.0, 3.0], mode="serial_sim")
    assert ok and row.split(",")[9] == ""  # simulate mode: no wall time
    for variant in ("paco", "const-pieces"):
        row, ok = cli.run_strassen(256, 7, variant=variant, gamma=1, mode="parallel")
        assert ok, row
    row, ok = cli.run_strassen(512, 8, base=64, split_leftover=True, mode="parallel")
    assert ok, row
    out = io.StringIO()
    assert cli.run_spec({"algo": "mm", "n": "64,96", "p": "1,2", "mode": "parallel"}, out)
    assert len(out.getvalue().strip().splitlines()) == 5

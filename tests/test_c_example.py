"""The C ABI from plain C (examples/c_minplus.c): compiles with gcc against
include/paco_b200.h and libpaco_b200.so, then (on a GPU) runs and must match the
defining sums for one launch and for a hand-driven 5-worker MM-1-Piece plan."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2011_01441_b200")


def _build(tmp_path):
    exe = tmp_path / "c_minplus"
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_minplus.c"), "-L", LIBDIR, "-lpaco_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libpaco_b200.so")):
        pytest.skip("library not built")
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    out = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("ok") == 2

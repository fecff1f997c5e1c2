"""The C-ABI library loads on a CPU-only host and exports every declared symbol."""

import ctypes
import os
import re

import pytest

from paper_2011_01441_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "paco_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(paco_[a-z0-9_]+)\s*\(", text)))


def test_all_header_symbols_exported_and_bound():
    lib = nat.load()
    names = header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
        assert name in nat.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.paco_abi_version() == 1


def test_tile_shapes():
    for sr in range(nat.SR_COUNT):
        bm, bn, bk, cps = nat.tile_shape(sr)
        assert bm > 0 and bn > 0 and bk > 0 and cps >= 1


def test_argument_errors_without_device():
    lib = nat.load()
    rc = lib.paco_mm(0, None, 99, None, 0, None, 0, None, 0, 1, 1, 1, None, 0, 0)
    assert rc == nat.ERR_ARG and b"semiring" in lib.paco_last_error()
    rc = lib.paco_mm(0, None, nat.SR_F32, None, 4, None, 4, None, 4, 4, 4, 4, None, 0, 0)
    assert rc == nat.ERR_ARG and b"null" in lib.paco_last_error()
    rc = lib.paco_mm(0, None, nat.SR_F32, 16, 2, 16, 4, 16, 4, 4, 4, 4, None, 0, 0)
    assert rc == nat.ERR_ARG and b"leading dimension" in lib.paco_last_error()
    with pytest.raises(ValueError):
        nat.check(rc)
    with pytest.raises(nat.PlanError):
        nat.plan_one_piece(1, 1, 1, 2)

"""SEMIRING_F64 on the FP64 tensor pipe (dmma_f64_kernel, one paco_mm launch):
against torch's f64 product (cuBLAS DGEMM) within 1e-12 relative, over aligned
and ragged shapes, partial k blocks, C accumulation, the PACO CTA plan (k-split
pieces folded with f64 atomics), explicit atomic folding and unaligned views."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(n, m, k, *, flags=0, overwrite=True, c0=None, a=None, b=None, seed=0):
    from paper_2011_01441_b200 import _native as nat
    from paper_2011_01441_b200.device import View
    from paper_2011_01441_b200.mm import launch_mm
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(n, k, device="cuda", dtype=torch.float64, generator=g) if a is None else a
    b = torch.randn(k, m, device="cuda", dtype=torch.float64, generator=g) if b is None else b
    c = (torch.zeros(n, m, device="cuda", dtype=torch.float64) if c0 is None else c0.clone())
    launch_mm(nat.SR_F64, torch.cuda.current_stream(), View.of(a), View.of(b), View.of(c), overwrite=overwrite,
              flags=flags)
    torch.cuda.synchronize()
    ref = a @ b + (0 if (c0 is None or overwrite) else c0)
    err = float((c - ref).norm() / ref.norm())
    return err


@pytest.mark.parametrize("shape", [(128, 128, 128), (300, 200, 77), (129, 257, 33), (1000, 1000, 1000),
                                   (2048, 1536, 4096), (64, 4096, 4100)])
def test_dmma_shapes(shape):
    assert _run(*shape) < 1e-12, shape


def test_dmma_accumulate_and_plans():
    from paper_2011_01441_b200 import _native as nat
    g = torch.Generator(device="cuda").manual_seed(3)
    c0 = torch.randn(1536, 1280, device="cuda", dtype=torch.float64, generator=g)
    assert _run(1536, 1280, 3000, overwrite=False, c0=c0) < 1e-12
    # PACO cuboid CTA plan: pieces cut k, their partial faces fold with f64 atomics
    assert _run(1536, 1280, 3000, overwrite=False, c0=c0, flags=nat.MM_PACO_PLAN) < 1e-12
    assert _run(4096, 4096, 2048, overwrite=True, flags=nat.MM_PACO_PLAN) < 1e-12
    # every tile folded atomically into C
    assert _run(777, 555, 999, overwrite=False, c0=torch.zeros(777, 555, device="cuda", dtype=torch.float64),
                flags=nat.MM_ATOMIC) < 1e-12


def test_dmma_views():
    g = torch.Generator(device="cuda").manual_seed(4)
    big_a = torch.randn(700, 901, device="cuda", dtype=torch.float64, generator=g)
    big_b = torch.randn(901, 650, device="cuda", dtype=torch.float64, generator=g)
    # 16-byte aligned views with a row pitch of whole 16-byte units (TMA path) ...
    assert _run(600, 500, 800, a=big_a[2:602, 4:804].contiguous()[:, :], b=big_b[:800, 6:506]) < 1e-12
    # ... and views off 16-byte alignment (odd row pitch: repacked or the element path)
    assert _run(600, 500, 800, a=big_a[1:601, 1:801], b=big_b[1:801, 1:501]) < 1e-12


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_dmma_mm_execute_plans(p):
    """The reference's executor on SEMIRING_F64: big COMPUTE cuboids leave the
    batched DFMA launch for one DMMA launch each; k-cut folds stay exact to 1e-12."""
    from paper_2011_01441_b200 import matmul as M
    g = torch.Generator(device="cuda").manual_seed(10 + p)
    n, m, k = 1536, 1280, 2048
    a = torch.randn(n, k, device="cuda", dtype=torch.float64, generator=g)
    b = torch.randn(k, m, device="cuda", dtype=torch.float64, generator=g)
    c = torch.randn(n, m, device="cuda", dtype=torch.float64, generator=g)
    want = c + a @ b
    for fused in (True, False):
        got = c.clone()
        M.mm_execute(M.mm_one_piece_partition(n, m, k, p), a, b, got, M.SEMIRING_F64, fused_folds=fused)
        torch.cuda.synchronize()
        assert float((got - want).norm() / want.norm()) < 1e-12, (p, fused)

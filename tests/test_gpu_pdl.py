"""Programmatic dependent launch with early operand loads (tc_gemm.cu pdl_track):
back-to-back resident-B tcgen05 launches load their first tile before
griddepcontrol.wait unless an operand may still be written by an in-flight
tcgen05 launch on the stream.  A launch reading the bytes its predecessor
writes must see them; independent launches stay exact."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _launch(a, b, c, st):
    from paper_2011_01441_b200 import _native as nat
    from paper_2011_01441_b200.device import View
    from paper_2011_01441_b200.mm import launch_mm
    launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)


def test_pdl_chain_reads_predecessor_output():
    st = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(1)
    n, k, m = 32768, 256, 1024
    # entries in {-1, 0, 1}: C1 holds integers |x| <= 256, whose f32 words have zero low
    # halves, so C1's bytes read as bf16 are finite (0, x, 0, x, ...)
    a1 = torch.randint(-1, 2, (n, k), device="cuda", generator=g).to(torch.bfloat16)
    b1 = torch.randint(-1, 2, (k, m), device="cuda", generator=g).to(torch.bfloat16)
    buf = torch.zeros(n * m, device="cuda", dtype=torch.float32)   # launch 1's C ...
    c1 = buf.view(n, m)
    # ... is launch 2's A (as bf16 bits): the last row blocks of column block 0, among
    # the tiles launch 1 writes last
    a2 = buf.view(torch.bfloat16).view(n, 2 * m)[n - 4096:, :256]
    b2 = torch.randn(256, 512, device="cuda", generator=g).to(torch.bfloat16)
    for rep in range(5):
        buf.zero_()
        c2 = torch.empty(4096, 512, device="cuda")
        _launch(a1, b1, c1, st)      # long: 32768 x 1024 outputs
        _launch(a2, b2, c2, st)      # reads the first rows of c1's bytes
        torch.cuda.synchronize()
        assert torch.isfinite(a2.float()).all() and a2.float().abs().max() > 0
        ref = a2.double() @ b2.double()
        assert float((c2.double() - ref).norm() / ref.norm()) < 1e-5, rep


def test_pdl_independent_back_to_back():
    st = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(2)
    ops = []
    for i in range(6):
        n = 8192 * (1 + i % 3)
        a = torch.randn(n, 256, device="cuda", generator=g).to(torch.bfloat16)
        b = torch.randn(256, 768, device="cuda", generator=g).to(torch.bfloat16)
        ops.append((a, b, torch.empty(n, 768, device="cuda")))
    for _ in range(3):
        for a, b, c in ops:
            c.fill_(float("nan"))
        torch.cuda.synchronize()
        for a, b, c in ops:      # no host sync and no other kernel in between
            _launch(a, b, c, st)
        torch.cuda.synchronize()
        for a, b, c in ops:
            ref = a.double() @ b.double()
            assert float((c.double() - ref).norm() / ref.norm()) < 1e-5

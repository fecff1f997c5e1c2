"""Small launches of every kernel family for compute-sanitizer (one tool per run):

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_cases.py [cases]

cases (default all): simt (tropical tile kernel, vector and element load paths,
bulk and element epilogues, explicit k-split pieces, batch kernel), tc (bf16
resident-B and streaming kinds, 3xTF32 presplit and multi-destination),
remote (mm_execute's fused remote-fold epilogue at system scope on one GPU),
elementwise (fold, fill, lincomb, split, narrow/widen, naive).  Results are
checked against the CPU oracle so a silent corruption fails too.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import cref
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import mm as MM
from paper_2011_01441_b200 import strassen as S
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

INF = 2**30
cases = sys.argv[1].split(",") if len(sys.argv) > 1 else ["simt", "tc", "remote", "elementwise"]
rng = np.random.default_rng(7)
st = torch.cuda.current_stream()


def trop(shape, inf=0.1):
    x = rng.integers(0, 2**20, shape, dtype=np.int32)
    x[rng.random(shape) < inf] = INF
    return x


if "simt" in cases:
    for (n, m, k, off) in ((256, 256, 320, 0), (130, 200, 97, 1)):
        A, B = trop((n, k + off)), trop((k, m + off))
        a, b = torch.from_numpy(A).cuda()[:, off:], torch.from_numpy(B).cuda()[:, off:]
        want = cref.mm(cref.SR_MINPLUS_SAT32, A[:, off:], B[:, off:], np.full((n, m), INF, np.int32))
        for pieces in (None, [(0, 0, 0, 2, 2, 4), (0, 0, 4, 2, 2, 76)]):
            c = torch.full((n, m), INF, dtype=torch.int32, device="cuda")
            launch_mm(nat.SR_MINPLUS_SAT32, st, View.of(a), View.of(b), View.of(c),
                      pieces=pieces if (n, m) == (256, 256) else None)
            assert np.array_equal(c.cpu().numpy(), want), ("simt", n, m, k, off, pieces)
    plan = M.mm_one_piece_partition(300, 260, 515, 5)   # batched launch with fused k-cut folds
    A, B = trop((300, 515)), trop((515, 260))
    C = np.full((300, 260), INF, np.int32)
    M.mm_execute(plan, A, B, C, M.SEMIRING_MINPLUS_SAT)
    assert np.array_equal(C, cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((300, 260), INF, np.int32)))
    print("simt ok")

if "tc" in cases:
    for (n, m, k) in ((512, 512, 256), (384, 640, 512)):
        a = torch.randn(n, k, device="cuda").to(torch.bfloat16)
        b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
        c = torch.empty(n, m, device="cuda")
        M.mm_seq(a, b, c, M.SEMIRING_BF16, overwrite=True)
        ref = a.double() @ b.double()
        assert float((c.double() - ref).norm() / ref.norm()) < 1e-5, ("bf16", n, m, k)
    x = torch.rand(512, 512, device="cuda") * 2 - 1
    y = torch.rand(512, 512, device="cuda") * 2 - 1
    z = torch.zeros(512, 512, device="cuda")
    M.mm_seq(x, y, z, M.SEMIRING_F32)
    ref = x.double() @ y.double()
    assert float((z.double() - ref).norm() / ref.norm()) < 1e-5
    C = S.strassen_seq(x, y, 512, base=128)   # 3xTF32 multi-destination leaves
    assert float((C.double() - ref).norm() / ref.norm()) < 1e-4
    print("tc ok")

if "remote" in cases:
    MM._REMOTE_ALL = "fused"
    A, B = trop((301, 603)), trop((603, 257))
    C0 = rng.integers(0, 2**21, (301, 257)).astype(np.int32)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy())
    for plan in (M.mm_one_piece_partition(301, 257, 603, 5), M.mm_paco_partition(301, 257, 603, 3, base=32)):
        C = C0.copy()
        M.mm_execute(plan, A, B, C, M.SEMIRING_MINPLUS_SAT, batch=False)
        assert np.array_equal(C, want)
    MM._REMOTE_ALL = ""
    print("remote ok")

if "elementwise" in cases:
    MM.NARROW_MIN_TERMS = 0
    A64 = rng.integers(0, 2**31, (70, 90), dtype=np.int64)
    B64 = rng.integers(0, 2**31, (90, 50), dtype=np.int64)
    C = np.full((70, 50), int(M.MINPLUS_INF), np.int64)
    M.mm_seq(A64, B64, C, M.SEMIRING_MINPLUS)
    assert np.array_equal(C, cref.mm(cref.SR_MINPLUS_I64, A64, B64, np.full((70, 50), int(M.MINPLUS_INF), np.int64)))
    d = M.mm_oracle(trop((33, 17)), trop((17, 29)), M.SEMIRING_MINPLUS_SAT)
    assert d.shape == (33, 29)
    C = np.full((300, 260), INF, np.int32)
    A, B = trop((300, 515)), trop((515, 260))
    M.mm_execute(M.mm_one_piece_partition(300, 260, 515, 7), A, B, C, M.SEMIRING_MINPLUS_SAT, fused_folds=False)
    assert np.array_equal(C, cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((300, 260), INF, np.int32)))
    print("elementwise ok")
torch.cuda.synchronize()
print("sanitize cases ok")

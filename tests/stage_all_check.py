"""Helper of tests/test_gpu_mm.py::test_remote_worker_paths (argv[1] = fused |
stage): every plan worker takes mm_execute's remote-GPU path on the single
test GPU (the product's test hooks mm._REMOTE_ALL / strassen._STAGE_ALL)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import cref
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import mm as _mm
from paper_2011_01441_b200 import strassen as _st

_mm._REMOTE_ALL = sys.argv[1]
_st._STAGE_ALL = True

rng = np.random.default_rng(71)
n, m, k = 301, 257, 603
A = rng.integers(0, 2**20, (n, k)).astype(np.int32)
B = rng.integers(0, 2**20, (k, m)).astype(np.int32)
C0 = rng.integers(0, 2**21, (n, m)).astype(np.int32)
want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy())
for p in (3, 5, 8):
    for plan in (M.mm_one_piece_partition(n, m, k, p), M.mm_paco_partition(n, m, k, p, base=32)):
        for fused in (None, False):
            for mode in ("serial_sim", "parallel"):
                C = C0.copy()
                M.mm_execute(plan, A, B, C, M.SEMIRING_MINPLUS_SAT, mode=mode, fused_folds=fused, batch=False)
                assert np.array_equal(C, want), (p, plan.meta["variant"], fused, mode)
Af = rng.uniform(-1, 1, (n, k)).astype(np.float32)
Bf = rng.uniform(-1, 1, (k, m)).astype(np.float32)
ref = Af.astype(np.float64) @ Bf.astype(np.float64)
for sem in (M.SEMIRING_F32, M.SEMIRING_F32_SIMT):
    C = np.zeros((n, m), np.float32)
    M.mm_execute(M.mm_paco_partition(n, m, k, 5, base=32), Af, Bf, C, sem, mode="parallel", batch=False)
    assert np.linalg.norm(C - ref) <= 1e-5 * np.linalg.norm(ref), sem.name
# Strassen plans: whole nodes and split-leaf pieces computed in "remote" local memory
from paper_2011_01441_b200 import strassen as S
ns = 256
Ai = rng.integers(-30, 30, (ns, ns)).astype(np.int64)
Bi = rng.integers(-30, 30, (ns, ns)).astype(np.int64)
for plan in (S.strassen_paco_partition(ns, 5, base=32, split_leftover=True),
             S.strassen_const_pieces_partition(ns, 6, S.SuperRoundCfg(2), base=32)):
    for mode in ("serial_sim", "parallel"):
        assert np.array_equal(S.strassen_execute(plan, Ai, Bi, mode), Ai @ Bi), (plan.meta["variant"], mode)
Af2 = rng.uniform(-1, 1, (ns, ns)).astype(np.float32)
Bf2 = rng.uniform(-1, 1, (ns, ns)).astype(np.float32)
Cf2 = S.strassen_execute(S.strassen_paco_partition(ns, 8, base=32, split_leftover=True), Af2, Bf2, "parallel")
ref2 = Af2.astype(np.float64) @ Bf2.astype(np.float64)
assert np.linalg.norm(Cf2 - ref2) <= 1e-4 * np.linalg.norm(ref2)
print("stage-all ok")

"""Multi-rank PACO-MM host logic on CPU with the gloo backend (world sizes 2 and 3).

The distributed executor (paper_2011_01441_b200/distributed.py) is run with a
CPU arithmetic double (the C oracle) so its task ownership, per-REDUCE process
groups, fold/reduce ordering and the one-holder invariant are exercised with
real collectives; the result must equal the single-process oracle exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cref
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200.distributed import DistributedMM

INF = 2**30
SR = {"minplus_sat": (M.SEMIRING_MINPLUS_SAT, cref.SR_MINPLUS_SAT32),
      "maxplus": (M.SEMIRING_MAXPLUS, cref.SR_MAXPLUS_SAT32),
      "int": (M.SEMIRING_INT, cref.SR_INT_I64)}


class CpuOps:
    """Test double of CudaOps: same interface, oracle arithmetic on CPU tensors."""

    def __init__(self, name):
        self.sr, self.cid = SR[name]
        self.name = name

    def combine(self, x, y):
        if self.name == "minplus_sat":
            return torch.minimum(x, y)
        if self.name == "maxplus":
            return torch.maximum(x, y)
        return x + y

    def compute(self, a, b, out):
        res = np.full(tuple(out.shape), self.sr.zero, dtype=self.sr.dtype)
        cref.mm(self.cid, a.numpy(), b.numpy(), res)
        out.copy_(self.combine(out, torch.from_numpy(res)))

    def fold(self, dst, src, reset):
        dst.copy_(self.combine(dst, src))
        if reset:
            src.fill_(int(self.sr.zero))

    def fill(self, dst):
        dst.fill_(int(self.sr.zero))

    def empty(self, shape, like):
        return torch.empty(shape, dtype=like.dtype)


def _inputs(name, n, m, k, seed):
    rng = np.random.default_rng(seed)
    if name == "minplus_sat":
        A = rng.integers(0, 2**20, (n, k), dtype=np.int32)
        A[rng.random(A.shape) < 0.1] = INF
        B = rng.integers(0, 2**20, (k, m), dtype=np.int32)
        B[rng.random(B.shape) < 0.1] = INF
        C = rng.integers(0, 2**21, (n, m), dtype=np.int32)
    elif name == "maxplus":
        A = rng.integers(-2**20, 2**20, (n, k), dtype=np.int32)
        B = rng.integers(-2**20, 2**20, (k, m), dtype=np.int32)
        C = np.full((n, m), -INF, np.int32)
    else:
        A = rng.integers(-50, 50, (n, k)).astype(np.int64)
        B = rng.integers(-50, 50, (k, m)).astype(np.int64)
        C = rng.integers(-1000, 1000, (n, m)).astype(np.int64)
    return A, B, C


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for idx, (name, variant, n, m, k) in enumerate(cases):
            A, B, C0 = _inputs(name, n, m, k, idx)
            plan = (M.mm_one_piece_partition(n, m, k, world) if variant == "one_piece"
                    else M.mm_paco_partition(n, m, k, world, base=8))
            ex = DistributedMM(plan, SR[name][0], CpuOps(name))
            C_local = torch.empty((n, m), dtype=torch.from_numpy(C0).dtype)
            ex.run(torch.from_numpy(A), torch.from_numpy(B), C_local, torch.from_numpy(C0))
            # every rank: the regions it claims to hold are final there
            ex.gather(C_local, dst=0)
            if rank == 0:
                want = cref.mm(SR[name][1], A, B, C0.copy())
                q.put((idx, bool(np.array_equal(C_local.numpy(), want)),
                       sum(1 for t in plan.tasks if t.kind == "reduce")))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_matches_oracle(world):
    cases = [
        ("minplus_sat", "one_piece", 16, 12, 200),   # k-heavy: forces k cuts -> reduces
        ("minplus_sat", "one_piece", 40, 30, 20),
        ("maxplus", "one_piece", 12, 10, 150),
        ("int", "one_piece", 10, 9, 120),
        ("minplus_sat", "paco", 33, 21, 47),         # multi-piece: nested temps/folds
        ("int", "paco", 24, 20, 60),
    ]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    results = sorted(q.get(timeout=5) for _ in cases)
    assert all(ok for _, ok, _ in results), results
    assert any(nred > 0 for _, _, nred in results)


@pytest.mark.parametrize("p", [2, 3, 5, 7, 8])
def test_fused_launches_cover_iteration_space_once(p):
    """Fused folds: all ranks' launches tile the (i, j, l) cuboid exactly once, and
    every launch writes inside one owner's rectangle of C."""
    from paper_2011_01441_b200.distributed import fused_launches
    rng = np.random.default_rng(p)
    for _ in range(6):
        n, m, k = (int(x) for x in rng.integers(8, 60, 3))
        for plan in (M.mm_one_piece_partition(n, m, k * 4, p), M.mm_paco_partition(n, m, k, p, base=6)):
            cover = np.zeros((plan.meta["n"], plan.meta["m"], plan.meta["k"]), np.int32)
            for r in range(p):
                owners, launches = fused_launches(plan, r)
                for (ai, al, an, ak), (bl, bj, bk, bm), owner, (ci, cj, cn, cm) in launches:
                    assert (an, bm) == (cn, cm) and ak == bk and al == bl
                    assert ci == ai and cj == bj  # C[i, j] gets A row i and B column j
                    cover[ai:ai + an, bj:bj + bm, al:al + ak] += 1
                    owner_rects = [o for o in owners if o[1] == owner]
                    assert any(o[0][0] <= ci and o[0][1] <= cj and ci + cn <= o[0][0] + o[0][2]
                               and cj + cm <= o[0][1] + o[0][3] for o in owner_rects)
            assert (cover == 1).all()


@pytest.mark.parametrize("shape,p", [((65536, 1024, 256), 2), ((65536, 1024, 256), 8), ((8192, 8192, 8192), 4),
                                     ((8192, 8192, 8192), 5), ((8192, 8192, 8192), 7), ((384, 320, 256), 3)])
def test_sole_writer_launches(shape, p):
    """FusedDistributedMM's store-only launches (PACO_MM_OVERWRITE: no zero fill,
    no atomics): exactly the local full-k launches whose C rectangle no other
    launch touches.  cfg3's n-only cuts make every launch one; a k-cut pair's
    two launches never are; sole rectangles tile what they cover once."""
    from paper_2011_01441_b200.distributed import _rect_intersect, fused_launches, sole_launches
    n, m, k = shape
    plan = M.mm_one_piece_partition(n, m, k, p) if shape != (384, 320, 256) else M.mm_paco_partition(n, m, k, p)
    nred = sum(1 for t in plan.tasks if t.kind == "reduce")
    covered = 0
    all_l = [(r, j, L) for r in range(p) for j, L in enumerate(fused_launches(plan, r)[1])]
    for r in range(p):
        launches = fused_launches(plan, r)[1]
        sole = sole_launches(plan, r)
        assert len(sole) == len(launches)
        for j, ((ai, al, an, ak), _, owner, rect) in enumerate(launches):
            others = [L for rr, jj, L in all_l if (rr, jj) != (r, j) and L[2] == owner and _rect_intersect(rect, L[3])]
            assert sole[j] == (owner == r and ak == k and not others)
            if sole[j]:
                covered += rect[2] * rect[3]
    if nred == 0:
        assert all(all(sole_launches(plan, r)) for r in range(p))
        assert covered == n * m
    else:
        assert covered < n * m

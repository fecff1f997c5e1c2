"""DistributedStrassen on the GPU: ranks as processes sharing the test box's one
GPU (no kernel waits on another rank), gloo for the reduce-scatter of the
signed partial C.  fp32 (3xTF32 leaves, 1e-4 relative Frobenius, the cfg5
tolerance) and the exact int64 ring, plain / split-leftover / const-pieces plans.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2011_01441_b200 import strassen as S
    from paper_2011_01441_b200.distributed import CudaStrassenOps, DistributedStrassen
    try:
        for n, base, variant, ring, seed in cases:
            rng = np.random.default_rng(seed)
            if ring == "f32":
                A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
                B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
                dt = torch.float32
            else:
                A = rng.integers(-1000, 1000, (n, n)).astype(np.int64)
                B = rng.integers(-1000, 1000, (n, n)).astype(np.int64)
                dt = torch.int64
            if variant == "const":
                plan = S.strassen_const_pieces_partition(n, world, S.SuperRoundCfg(1), base=base)
            else:
                plan = S.strassen_paco_partition(n, world, base=base, split_leftover=variant == "split")
            size = plan.meta["n_padded"]
            a = torch.zeros((size, size), dtype=dt, device="cuda")
            b = torch.zeros((size, size), dtype=dt, device="cuda")
            a[:n, :n] = torch.from_numpy(A)
            b[:n, :n] = torch.from_numpy(B)
            ds = DistributedStrassen(plan, CudaStrassenOps(dt))
            C = ds.gather(ds.run(a, b))
            if rank == 0:
                C = C.cpu().numpy()
                if ring == "f32":
                    ref = A.astype(np.float64) @ B.astype(np.float64)
                    ok = float(np.linalg.norm(C - ref) / np.linalg.norm(ref)) <= 1e-4
                else:
                    ok = bool(np.array_equal(C, A @ B))
                q.put(((n, base, variant, ring), ok, len(ds.pieces)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_strassen_gpu(world):
    cases = [(512, 64, "split", "f32", 1), (1000, 128, "paco", "f32", 2), (256, 32, "split", "i64", 3),
             (384, 32, "const", "i64", 4)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=5) for _ in cases]
    assert all(r[1] for r in res), res


def _raw_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2011_01441_b200 import strassen as S
    from paper_2011_01441_b200.distributed import CudaStrassenOps, DistributedStrassen
    calls = []
    name = "_leaf_level_b3" if S.LEAF_BF16X3 else "_leaf_level_b2raw"   # the single-GPU default leaves
    leaf = getattr(S, name)

    def counted(*a, **k):
        calls.append(1)
        return leaf(*a, **k)

    setattr(S, name, counted)
    try:
        n, base = 8192, 2048
        g = torch.Generator(device="cuda").manual_seed(7)
        a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
        b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
        plan = S.strassen_paco_partition(n, world, base=base)
        ds = DistributedStrassen(plan, CudaStrassenOps(torch.float32))
        C = ds.gather(ds.run(a, b))
        n_calls = [None] * world
        dist.all_gather_object(n_calls, len(calls))
        if rank == 0:
            rows = torch.arange(0, n, 97, device="cuda")
            ref = a[rows].double() @ b.double()
            err = float((C[rows].double() - ref).norm() / ref.norm())
            q.put((err, n_calls))
    finally:
        dist.destroy_process_group()


def test_distributed_strassen_raw_leaves():
    """Rank nodes big enough for the CTA-pair batch take the same leaves as the
    single-GPU path (strassen.strassen_into: bf16x3, or the raw-operand tf32 +
    2 x bf16 format)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_raw_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    err, n_calls = q.get(timeout=5)
    assert err <= 1e-4, err
    assert all(c >= 1 for c in n_calls), n_calls


def test_strassen_into_leaf_raw_pair():
    """A rank's leaf-sized node (n <= base) with signed placements: one CTA-pair
    product on raw fp32 operands folded +/- into two C blocks."""
    from paper_2011_01441_b200 import strassen as S
    from paper_2011_01441_b200.device import View
    n = 4096
    g = torch.Generator(device="cuda").manual_seed(11)
    a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    C = torch.rand(n, 2 * n, device="cuda", generator=g)
    C0 = C.clone()
    st = torch.cuda.current_stream()
    assert S.strassen_into(View.of(a), View.of(b), [(View.of(C[:, :n]), 1), (View.of(C[:, n:]), -1)], n, st)
    rows = torch.arange(0, n, 61, device="cuda")
    ref = a[rows].double() @ b.double()
    for half, sg in ((0, 1), (1, -1)):
        got = C[rows, half * n:(half + 1) * n].double() - C0[rows, half * n:(half + 1) * n].double()
        err = float((got - sg * ref).norm() / ref.norm())
        assert err <= 1e-4, (half, err)

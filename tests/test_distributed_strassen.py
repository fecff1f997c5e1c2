"""Multi-rank Strassen executor host logic on CPU with gloo (world sizes 2, 3, 5).

``DistributedStrassen`` (paper_2011_01441_b200/distributed.py) is run with a
CPU arithmetic double (exact int64 NumPy products as leaves, the Strassen
recursion of each node restated by the oracle) so its per-rank operand
formation, the signed placement of every node product / split-leaf piece in C
and the reduce-scatter are exercised with real collectives; the gathered C
must equal A @ B exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import paco_numpy as ref
from paper_2011_01441_b200 import strassen as S
from paper_2011_01441_b200.distributed import DistributedStrassen, strassen_placements


class CpuStrassenOps:
    """Test double of CudaStrassenOps on CPU int64 tensors."""

    def zeros(self, shape, like):
        return torch.zeros(shape, dtype=like.dtype)

    def lincomb(self, out, terms, accumulate):
        acc = out.clone() if accumulate else torch.zeros_like(out)
        for c, t in terms:
            acc += c * t
        out.copy_(acc)

    def strassen(self, a, b, out, base):
        levels = max(0, (a.shape[0] // base).bit_length() - 1)
        out.copy_(torch.from_numpy(ref.strassen(a.numpy(), b.numpy(), levels)))

    def mm(self, a, b, out):
        out.copy_(torch.from_numpy(a.numpy() @ b.numpy()))


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for n, base, variant, seed in cases:
            rng = np.random.default_rng(seed)
            A = rng.integers(-20, 20, (n, n)).astype(np.int64)
            B = rng.integers(-20, 20, (n, n)).astype(np.int64)
            if variant == "split":
                plan = S.strassen_paco_partition(n, world, base=base, split_leftover=True)
            elif variant == "const":
                plan = S.strassen_const_pieces_partition(n, world, S.SuperRoundCfg(1), base=base)
            else:
                plan = S.strassen_paco_partition(n, world, base=base)
            size = plan.meta["n_padded"]
            a = torch.zeros((size, size), dtype=torch.int64)
            b = torch.zeros((size, size), dtype=torch.int64)
            a[:n, :n] = torch.from_numpy(A)
            b[:n, :n] = torch.from_numpy(B)
            ds = DistributedStrassen(plan, CpuStrassenOps())
            slab = ds.run(a, b)
            C = ds.gather(slab)
            if rank == 0:
                q.put(((n, base, variant), bool(np.array_equal(C.numpy(), A @ B))))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3, 5])
def test_distributed_strassen_exact(world):
    cases = [(32, 4, "paco", 1), (32, 4, "split", 2), (64, 8, "split", 3), (40, 4, "const", 4), (16, 2, "paco", 5)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in cases]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in got), got


def test_placements_reconstruct_one_level():
    """Signed placements of the seven depth-1 products rebuild C exactly."""
    rng = np.random.default_rng(0)
    A = rng.integers(-9, 9, (8, 8)).astype(np.int64)
    B = rng.integers(-9, 9, (8, 8)).astype(np.int64)
    C = np.zeros((8, 8), np.int64)
    h = 4

    def quad(X, q):
        return X[int(q[0]) * h:(int(q[0]) + 1) * h, int(q[1]) * h:(int(q[1]) + 1) * h]

    for r in range(1, 8):
        s = sum(c * quad(A, q) for c, q in S.S_TERMS[r])
        t = sum(c * quad(B, q) for c, q in S.T_TERMS[r])
        for sign, i, j in strassen_placements((r,), 8):
            C[i:i + h, j:j + h] += sign * (s @ t)
    assert np.array_equal(C, A @ B)
    # each M_r appears once per occurrence in the C-block formulas: 12 in total
    assert sum(len(strassen_placements((r,), 8)) for r in range(1, 8)) == 12
    assert len(strassen_placements((1, 1), 16)) == 4

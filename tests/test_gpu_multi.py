"""Cross-GPU paths on real NVLink -- run only on a box with 2+ GPUs (skipped otherwise).

The single-GPU suite covers these executors with ranks co-scheduled on one
device; here the folds really cross NVLink: mm_execute(devices=[0, 1]) with a
k-cut plan (a worker on GPU 1 folds its tiles into GPU 0's C with system-scope
atomics, tcgen05 workers through staged copies), and FusedDistributedMM with one
process per GPU over NCCL (stream-ordered fold handshake, remote IPC folds).
Bit-exact against the CPU oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs 2+ GPUs (NVLink peers)")]
INF = 2**30


def _inputs(n, m, k, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(0, 2**20, (n, k), dtype=np.int32)
    A[rng.random(A.shape) < 0.1] = INF
    B = rng.integers(0, 2**20, (k, m), dtype=np.int32)
    B[rng.random(B.shape) < 0.1] = INF
    return A, B


def test_mm_execute_two_devices_k_cut():
    from oracle import cref
    from paper_2011_01441_b200 import matmul as M
    n = m = k = 1536
    A, B = _inputs(n, m, k, 1)
    want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((n, m), INF, np.int32))
    for p in (5, 7):   # MM-1-Piece cuts k at p = 5 (1 pair) and 7 (3 pairs)
        plan = M.mm_one_piece_partition(n, m, k, p)
        assert any(t.kind == "reduce" for t in plan.tasks)
        for fused in (True, False):
            C = np.full((n, m), INF, np.int32)
            M.mm_execute(plan, A, B, C, M.SEMIRING_MINPLUS_SAT, mode="parallel", devices=[0, 1],
                         fused_folds=fused)
            assert np.array_equal(C, want), (p, fused)
    # tcgen05 workers on the second GPU: staged blocks folded on the home GPU
    a = torch.randn(1024, 512, device="cuda:0").to(torch.bfloat16)
    b = torch.randn(512, 768, device="cuda:0").to(torch.bfloat16)
    c = torch.zeros(1024, 768, device="cuda:0")
    M.mm_execute(M.mm_one_piece_partition(1024, 768, 512, 5), a, b, c, M.SEMIRING_BF16, devices=[0, 1])
    ref = a.double() @ b.double()
    assert float((c.double() - ref).norm() / ref.norm()) < 1e-5


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2011_01441_b200 import _native as nat
    from paper_2011_01441_b200 import matmul as M
    from paper_2011_01441_b200.distributed import FusedDistributedMM
    from paper_2011_01441_b200.mm import _copy2d_raw
    try:
        n = m = k = 1536
        A, B = _inputs(n, m, k, 2)
        plan = M.mm_one_piece_partition(n, m, k, world)
        for style in ("atomic", "stage"):
            ex = FusedDistributedMM(plan, M.SEMIRING_MINPLUS_SAT, nat.SR_MINPLUS_SAT32, rank, fold_style=style)
            for _ in range(2):   # the second step re-runs the handshakes over the same buffers
                ex.run(torch.from_numpy(A).cuda(rank), torch.from_numpy(B).cuda(rank))
            mine = torch.empty((n, m), dtype=torch.int32, device=f"cuda:{rank}")
            _copy2d_raw(rank, mine, ex.own_ptr, m * 4)
            host = mine.cpu().numpy()
            pieces = [(r, host[r[0]:r[0] + r[2], r[1]:r[1] + r[3]].copy()) for r in ex.owned]
            allp = [None] * world
            dist.all_gather_object(allp, pieces)
            dist.barrier()
            ex.close()
            if rank == 0:
                from oracle import cref
                C = np.full((n, m), -1, np.int32)
                for plist in allp:
                    for (i0, j0, rn, rm), blk in plist:
                        C[i0:i0 + rn, j0:j0 + rm] = blk
                want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, np.full((n, m), INF, np.int32))
                q.put((style, bool(np.array_equal(C, want)), ex.exchange))
    finally:
        dist.destroy_process_group()


def test_fused_distributed_across_gpus():
    world = min(torch.cuda.device_count(), 5)   # 5 ranks cut k when the box has them
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=5) for _ in range(2)]
    assert all(ok for _, ok, _ in res), res

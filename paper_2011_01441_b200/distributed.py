"""Multi-GPU PACO-MM: one process per GPU, plan worker == rank.

The GPU level of the two-level PACO scheme: the cuboid is cut
with the reference partitioners (mm_one_piece_partition / mm_paco_partition /
mm_hetero_partition, matmul.py:214-339) for p = world_size; each rank runs its
COMPUTE tasks with the sm_100a kernels (and the CTA-level plan inside), and the
only data exchange is the plan's REDUCE tasks -- the fold of a k-cut's
temporary into its sibling's C face (matmul.py:455-460), done here as an NCCL
reduction with the semiring's (+) (MIN / MAX / SUM) over the reduce's workers.

Invariant that makes any plan correct: every element of every buffer has
exactly one holder rank; all other ranks keep the semiring zero there.  A
REDUCE over workers G then (1) folds the target region into the temp locally
and zeroes the region, (2) reduces the temp onto G's first worker, and (3)
that worker folds the temp back into the region while the others zero the
temp -- the holder moves to G[0] exactly like the reference runs a REDUCE on
its first worker (core.py:301-303).

The arithmetic is pluggable (``ops``) so the host logic is testable with the
gloo backend on CPU; the product path uses ``CudaOps`` (sm_100a kernels).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .cuboid import temp_shape
from .plan import COMPUTE, REDUCE, Plan, PlanError

_REDUCE_OPS = {
    "int": dist.ReduceOp.SUM, "f64": dist.ReduceOp.SUM, "f32": dist.ReduceOp.SUM,
    "bf16": dist.ReduceOp.SUM, "minplus": dist.ReduceOp.MIN, "minplus_sat": dist.ReduceOp.MIN,
    "maxplus": dist.ReduceOp.MAX,
}


class CudaOps:
    """Device arithmetic for the distributed executor (sm_100a kernels)."""

    def __init__(self, semiring, kernel_id: int, stream: torch.cuda.Stream | None = None):
        self.semiring = semiring
        self.kid = kernel_id
        self.stream = stream

    def _st(self, t: torch.Tensor):
        return self.stream or torch.cuda.current_stream(t.device)

    def compute(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
        from .device import View
        from .mm import launch_mm

        launch_mm(self.kid, self._st(out), View.of(a), View.of(b), View.of(out))

    def fold(self, dst: torch.Tensor, src: torch.Tensor, reset: bool) -> None:
        from .device import View
        from .mm import launch_fold

        launch_fold(self.semiring.kernel_id, self._st(dst), View.of(dst), View.of(src), reset)

    def fill(self, dst: torch.Tensor) -> None:
        from .device import View
        from .mm import launch_fill

        launch_fill(self.semiring.kernel_id, self._st(dst), View.of(dst))

    def empty(self, shape, like: torch.Tensor) -> torch.Tensor:
        return torch.empty(shape, dtype=like.dtype, device=like.device)


@dataclass
class _Fold:
    task_id: int
    workers: tuple[int, ...]
    group: object
    temp: int
    target: int
    region: tuple[int, int, int, int]


class DistributedMM:
    """Execute one plan across ``world_size`` ranks (plan.p must equal it).

    Construct on every rank in the same order (it creates one process group
    per multi-rank REDUCE).  ``run`` is then called with this rank's operands.
    """

    def __init__(self, plan: Plan, semiring, ops, *, group=None):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if plan.p != self.world:
            raise PlanError(f"plan built for p={plan.p}, world size is {self.world}")
        plan.validate()
        self.plan = plan
        self.semiring = semiring
        self.ops = ops
        self.op = _REDUCE_OPS[semiring.name]
        self.folds: list[_Fold] = []
        for t in plan.tasks:
            if t.kind != REDUCE:
                continue
            ws = t.workers()
            grp = dist.new_group(list(ws)) if len(ws) > 1 else None
            bid, tgt, oi, oj, n, m = plan.meta["reduces"][t.id]
            self.folds.append(_Fold(t.id, ws, grp, bid, tgt, (oi, oj, n, m)))
        self._fold_at = {f.task_id: f for f in self.folds}
        self.mine = [t for t in plan.tasks if t.kind == COMPUTE and t.worker == self.rank]
        need = {t.region.out for t in self.mine if t.region.out}
        need |= {f.temp for f in self.folds if self.rank in f.workers}
        self.temp_ids = sorted(need)

    def owned_regions(self) -> list[tuple[int, int, int, int]]:
        """C rectangles (i0, j0, n, m) this rank holds after ``run``."""
        regions = []
        for t in self.mine:
            if t.region.out == 0:
                regions.append((t.region.out_i0, t.region.out_j0, t.region.n, t.region.m))
        moved = {}
        for f in self.folds:
            if f.target == 0:
                moved[f.region] = f.workers[0]
        keep = [r for r in regions if moved.get(r, self.rank) == self.rank]
        keep += [r for r, w in moved.items() if w == self.rank and r not in keep]
        return keep

    def run(self, A: torch.Tensor, B: torch.Tensor, C_local: torch.Tensor,
            C_init: torch.Tensor | None = None) -> None:
        """Compute this rank's share into ``C_local`` (full n x m, this rank's copy).

        ``C_init`` (the caller's C) is folded in for the regions of this rank's
        out=0 tasks; every other element of ``C_local`` starts at zero.
        """
        ops = self.ops
        ops.fill(C_local)
        if C_init is not None:
            for t in self.mine:
                c = t.region
                if c.out == 0:
                    ops.fold(C_local[c.out_i0:c.out_i0 + c.n, c.out_j0:c.out_j0 + c.m],
                             C_init[c.out_i0:c.out_i0 + c.n, c.out_j0:c.out_j0 + c.m], False)
        temps = {}
        for bid in self.temp_ids:
            temps[bid] = ops.empty(temp_shape(self.plan, bid), C_local)
            ops.fill(temps[bid])

        def buf(bid):
            return C_local if bid == 0 else temps[bid]

        for t in self.plan.tasks:
            if t.kind == COMPUTE:
                if t.worker != self.rank:
                    continue
                c = t.region
                out = buf(c.out)[c.out_i0:c.out_i0 + c.n, c.out_j0:c.out_j0 + c.m]
                ops.compute(A[c.i0:c.i0 + c.n, c.l0:c.l0 + c.k], B[c.l0:c.l0 + c.k, c.j0:c.j0 + c.m], out)
            elif t.kind == REDUCE:
                f = self._fold_at[t.id]
                if self.rank not in f.workers:
                    continue
                oi, oj, n, m = f.region
                region = buf(f.target)[oi:oi + n, oj:oj + m]
                tmp = temps[f.temp]
                if f.group is None:  # single-worker reduce: purely local
                    ops.fold(region, tmp, True)
                    continue
                ops.fold(tmp, region, True)           # (1) temp (+)= region; region = zero
                dist.reduce(tmp, dst=f.workers[0], op=self.op, group=f.group)  # (2)
                if self.rank == f.workers[0]:
                    ops.fold(region, tmp, True)       # (3) holder moves to the first worker
                else:
                    ops.fill(tmp)

    def gather(self, C_local: torch.Tensor, dst: int = 0) -> None:
        """Assemble the full C on ``dst``: one (+)-reduce of the holder copies."""
        dist.reduce(C_local, dst=dst, op=self.op)

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


def fused_launches(plan: Plan, rank: int):
    """Owner map and this rank's kernel launches for fused folds.

    Owners: the out=0 COMPUTE rectangles (they partition C) with their worker.
    Launches: every COMPUTE task of ``rank`` whose final C rectangle (temps
    resolved through the REDUCE chain, ``mm.fold_destinations``) is cut along
    the owner rectangles it overlaps: (A rows/cols, B rows/cols, owner, C rect).
    """
    from .mm import fold_destinations

    owners = []
    for t in plan.tasks:
        if t.kind == COMPUTE and t.region.out == 0:
            c = t.region
            owners.append(((c.out_i0, c.out_j0, c.n, c.m), t.worker))
    dest = fold_destinations(plan)
    launches = []
    for t in plan.tasks:
        if t.kind != COMPUTE or t.worker != rank:
            continue
        c = t.region
        _, fi, fj = dest.get(c.out, (0, 0, 0))
        D = (fi + c.out_i0, fj + c.out_j0, c.n, c.m)
        for rect, owner in owners:
            x = _rect_intersect(D, rect)
            if x is None:
                continue
            di, dj = x[0] - D[0], x[1] - D[1]
            launches.append(((c.i0 + di, c.l0, x[2], c.k), (c.l0, c.j0 + dj, c.k, x[3]), owner, x))
    return owners, launches


def sole_launches(plan: Plan, rank: int) -> list[bool]:
    """Per launch of ``rank`` (``fused_launches`` order): does it alone write its
    C rectangle -- local owner, the whole k extent, and no other launch of any
    rank folding into an intersecting rectangle of the same owner?"""
    k_all = plan.meta["k"]
    mine = fused_launches(plan, rank)[1]
    every = [(r, jj, o, rr) for r in range(plan.p) for jj, (_, _, o, rr) in enumerate(fused_launches(plan, r)[1])]
    return [owner == rank and a[3] == k_all and not any(
        (r, jj) != (rank, j) and o == owner and _rect_intersect(rect, rr) for r, jj, o, rr in every)
        for j, (a, _, owner, rect) in enumerate(mine)]


def _rect_intersect(a, b):
    i0, j0 = max(a[0], b[0]), max(a[1], b[1])
    i1, j1 = min(a[0] + a[2], b[0] + b[2]), min(a[1] + a[3], b[1] + b[3])
    return (i0, j0, i1 - i0, j1 - j0) if i1 > i0 and j1 > j0 else None


class FusedDistributedMM:
    """One process per GPU with the k-cut folds fused into the kernels.

    Every C element is owned by the rank whose out=0 COMPUTE task covers it
    (those rectangles partition C).  Each rank's C lives in IPC-shareable
    device memory; a task whose output is a temporary writes its tiles
    straight to their final place in the owners' C -- over NVLink for remote
    owners (element atomics, ``PACO_MM_REMOTE``), locally with the TMA bulk
    reduction -- so the plan's REDUCE tasks vanish: no temporaries, no fold
    pass, no NCCL call on the data path.  Remote folds use the TMA bulk
    reduction too when ``remote_bulk=True`` and a start-up probe shows it
    lands correctly in peer memory (``remote_bulk``).  Construct on every rank (it exchanges IPC
    handles with ``all_gather_object``).
    """

    def __init__(self, plan: Plan, semiring, kernel_id: int, device: int, *, group=None,
                 fold_style: str = "atomic", remote_bulk: bool = False, fold_probe: bool = True):
        import ctypes
        import os

        import numpy as np

        from . import _native as nat
        from .device import View, torch_dtype
        from .mm import fold_destinations

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if plan.p != self.world:
            raise PlanError(f"plan built for p={plan.p}, world size is {self.world}")
        plan.validate()
        self.plan, self.semiring, self.kid, self.device, self.group = plan, semiring, kernel_id, device, group
        self.n, self.m = plan.meta["n"], plan.meta["m"]
        self.tdtype = torch_dtype(semiring.dtype)
        self.itemsize = np.dtype(semiring.dtype).itemsize
        self.op = _REDUCE_OPS[semiring.name]
        self.nat = nat
        lib = nat.load()
        ptr = ctypes.c_void_p()
        nat.check(lib.paco_device_alloc(device, self.n * self.m * self.itemsize, ctypes.byref(ptr)))
        self.own_ptr = ptr.value
        handle = ctypes.create_string_buffer(64)
        nat.check(lib.paco_ipc_handle(device, self.own_ptr, handle))
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=group)
        self.ptrs = []
        for r, h in enumerate(handles):
            if r == self.rank:
                self.ptrs.append(self.own_ptr)
                continue
            p = ctypes.c_void_p()
            nat.check(lib.paco_ipc_open(device, ctypes.create_string_buffer(h, 64), ctypes.byref(p)))
            self.ptrs.append(p.value)
        self.views = [View.raw(p, self.n, self.m, self.itemsize, device) for p in self.ptrs]
        owners, self.launches = fused_launches(plan, self.rank)
        self.owned = [rect for rect, w in owners if w == self.rank]
        # no rank writes into another's C (p <= 4 on a cube: no k cut): the
        # ranks are independent and a step needs no barrier at all
        self.exchange = any(o != r for r in range(self.world) for _, _, o, _ in fused_launches(plan, r)[1])
        # remote folds: "atomic" (default) = the kernel's epilogue folds each
        # finished tile straight into the owner's C over NVLink (element atomics,
        # or TMA bulk reductions with remote_bulk=True) -- compute and transfer
        # overlap tile by tile, ~1/p of C spread over the whole kernel; "stage" =
        # compute into a local temporary, one bulk copy into a staging slot in the
        # owner's memory (IPC), the owner folds it after a barrier.
        self.fold_style = fold_style
        if self.fold_style not in ("stage", "atomic"):
            raise ValueError(f"fold_style must be 'stage' or 'atomic', got {self.fold_style!r}")
        from .mm import _TC_KERNELS
        if kernel_id in _TC_KERNELS:
            # the tcgen05 epilogue folds only into local C (TMA reduce-add): a
            # remote owner's share goes through a staged block
            self.fold_style = "stage"
        if self.fold_style == "atomic" and self.exchange and not self._probe_remote(self.nat.MM_ATOMIC |
                                                                                   self.nat.MM_REMOTE):
            # the element atomics into a peer's IPC-mapped C did not land right on this
            # fabric (checked once, on every rank): staged folds need only peer copies
            self.fold_style = "stage"
        self.fold_probe_ms = None   # [[fused, staged] ms per rank] when the timing probe ran
        if self.fold_style == "atomic" and self.exchange and fold_probe and not self._atomic_folds_pay():
            self.fold_style = "stage"
        self.remote_bulk = self._probe_remote_bulk() if self.fold_style == "atomic" and remote_bulk else False
        # C rectangles of mine that another rank folds into over NVLink: the
        # owner's own folds there must be atomic w.r.t. the peer's at system
        # scope too, so those launches use system-scope element atomics
        # (MM_REMOTE semantics on local memory) -- or, when remote folds are TMA
        # bulk reductions, the same bulk path with system-scope element edges
        incoming_rects = [rect for r in range(self.world) if r != self.rank
                          for _, _, o, rect in fused_launches(plan, r)[1] if o == self.rank]
        self.shared = [owner == self.rank and self.fold_style == "atomic"
                       and any(_rect_intersect(rect, ir) for ir in incoming_rects)
                       for _, _, owner, rect in self.launches]
        # sole writers: a local launch over the whole k whose C rectangle no other
        # launch (of any rank) touches computes its block with a plain store
        # (PACO_MM_OVERWRITE) -- no zero fill, no atomics, C written once (the
        # n-only cuts of cfg3's skinny shape make every launch one)
        self.sole = sole_launches(plan, self.rank)
        sole_rects = {tuple(rect) for s_, (_, _, _, rect) in zip(self.sole, self.launches) if s_}
        self.fill_rects = [r for r in self.owned if tuple(r) not in sole_rects]
        self._nccl = dist.get_backend(group) == "nccl"
        self._tok = torch.zeros(1, dtype=torch.int32, device=device) if self._nccl else None
        self._setup_staging()

    def _setup_staging(self) -> None:
        """Staging slots: every rank's remote launches into this rank's C get a slot
        in one IPC buffer here; senders keep a local temporary per remote launch."""
        import ctypes

        from .device import View

        lib = self.nat.load()
        self.incoming = []   # (rect, offset in elements) of slots others fill
        self.outgoing = []   # per launch index: (slot offset at the owner) or None
        self.temps = {}
        self.stage_ptr = None
        self.stage_ptrs = [None] * self.world
        if self.fold_style != "stage" or self.world == 1:
            return
        slots = {}  # (src rank, launch index) -> offset at the owner
        sizes = [0] * self.world
        for r in range(self.world):
            for j, (_, _, owner, rect) in enumerate(fused_launches(self.plan, r)[1]):
                if owner == r:
                    continue
                slots[(r, j)] = sizes[owner]
                if owner == self.rank:
                    self.incoming.append((rect, sizes[owner]))
                sizes[owner] += rect[2] * rect[3]
        if sizes[self.rank]:
            ptr = ctypes.c_void_p()
            self.nat.check(lib.paco_device_alloc(self.device, sizes[self.rank] * self.itemsize, ctypes.byref(ptr)))
            self.stage_ptr = ptr.value
        handle = ctypes.create_string_buffer(64)
        if self.stage_ptr is not None:
            self.nat.check(lib.paco_ipc_handle(self.device, self.stage_ptr, handle))
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw if self.stage_ptr is not None else None, group=self.group)
        for r, h in enumerate(handles):
            if r == self.rank:
                self.stage_ptrs[r] = self.stage_ptr
            elif h is not None and any(o == r for _, _, o, _ in self.launches):
                p = ctypes.c_void_p()
                self.nat.check(lib.paco_ipc_open(self.device, ctypes.create_string_buffer(h, 64), ctypes.byref(p)))
                self.stage_ptrs[r] = p.value
        for j, (_, _, owner, rect) in enumerate(self.launches):
            if owner == self.rank:
                self.outgoing.append(None)
                continue
            self.outgoing.append(slots[(self.rank, j)])
            self.temps[j] = torch.empty((rect[2], rect[3]), dtype=self.tdtype, device=self.device)

    def _probe_remote_bulk(self) -> bool:
        """Can the TMA bulk-reduce epilogue fold into a peer's IPC-mapped C?

        Off unless asked for (remote_bulk=True): a TMA bulk reduction that the
        fabric rejected would leave a sticky CUDA error, and element atomics
        over NVLink are always legal for peer-mapped memory.  If it fails,
        remote folds use element atomics (MM_REMOTE)."""
        return self._probe_remote(self.nat.MM_ATOMIC, small=False)

    def _atomic_folds_pay(self, size: int = 1024, slack: float = 1.15) -> bool:
        """Measure, don't guess: is a block computed with its fold fused into a
        peer's C (element atomics over the fabric) faster than the staged form
        (local product, one peer copy, a fold)?  Every rank times both on a
        size x size x size block of its neighbour's C at the same time (so the
        links carry the real pattern), best of 3; the fused form is kept unless
        the slowest rank's fused time exceeds ``slack`` x its staged time."""
        from .device import View
        from .mm import launch_fill, launch_fold, launch_mm

        if self.world == 1 or self.n < size or self.m < size or self.itemsize != 4:
            return True
        dev = self.device
        st = torch.cuda.current_stream(dev)
        kid = self.nat.SR_MINPLUS_SAT32
        g = torch.Generator(device="cpu").manual_seed(4321)
        a = torch.randint(0, 2**20, (size, size), generator=g, dtype=torch.int32).to(dev)
        b = torch.randint(0, 2**20, (size, size), generator=g, dtype=torch.int32).to(dev)
        tmp = torch.empty((size, size), dtype=torch.int32, device=dev)
        ld = self.m * self.itemsize // 4
        peer = (self.rank + 1) % self.world
        pv = View.raw(self.ptrs[peer], size, size, 4, dev, ld=ld)
        mine = View.raw(self.own_ptr, size, size, 4, dev, ld=ld)

        def fused():
            launch_mm(kid, st, View.of(a), View.of(b), pv, flags=self.nat.MM_ATOMIC | self.nat.MM_REMOTE, device=dev)

        def staged():
            launch_mm(kid, st, View.of(a), View.of(b), View.of(tmp), overwrite=True, device=dev)
            self.nat.check(self.nat.load().paco_copy2d(dev, st.cuda_stream, self.ptrs[peer], ld * 4,
                                                       tmp.data_ptr(), size * 4, size * 4, size))
            launch_fold(kid, st, mine, View.of(tmp), False)   # the owner's fold, same size

        times = []
        for fn in (fused, staged):
            best = float("inf")
            for _ in range(4):
                torch.cuda.synchronize(dev)
                dist.barrier(group=self.group)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            times.append(best)
        launch_fill(kid, st, mine)   # leave this rank's probe block at the semiring zero
        torch.cuda.synchronize(dev)
        allt = [None] * self.world
        dist.all_gather_object(allt, times, group=self.group)
        dist.barrier(group=self.group)
        self.fold_probe_ms = allt
        return max(t[0] for t in allt) <= slack * max(t[1] for t in allt)

    def _probe_remote(self, flags: int, small: bool = True) -> bool:
        """Does a fold with ``flags`` into a peer's IPC-mapped C land right?

        Each rank folds a small known product into the next rank's buffer,
        every owner checks what landed against a local computation, and the
        answer is True only if all ranks agree (collective: call on every rank).
        """
        from .device import View
        from .mm import launch_fill, launch_mm

        if self.world == 1 or self.n < 128 or self.m < 128:
            return self.world == 1 or small  # no room to probe: ``small`` is the answer
        dev = self.device
        st = torch.cuda.current_stream(dev)
        g = torch.Generator(device="cpu").manual_seed(1234)
        a = torch.randint(0, 1000, (128, 8), generator=g, dtype=torch.int32).to(dev)
        b = torch.randint(0, 1000, (8, 128), generator=g, dtype=torch.int32).to(dev)
        probe_sr = self.nat.SR_MINPLUS_SAT32
        mine = View.raw(self.own_ptr, 128, 128, 4, dev, ld=self.m * self.itemsize // 4)
        launch_fill(probe_sr, st, mine)
        torch.cuda.synchronize(dev)
        dist.barrier(group=self.group)
        peer = (self.rank + 1) % self.world
        pv = View.raw(self.ptrs[peer], 128, 128, 4, dev, ld=self.m * self.itemsize // 4)
        ok = True
        try:
            launch_mm(probe_sr, st, View.of(a), View.of(b), pv, flags=flags, device=dev)
            torch.cuda.synchronize(dev)
        except Exception:
            ok = False
        dist.barrier(group=self.group)
        ref = torch.full((128, 128), 2**30, dtype=torch.int32, device=dev)
        launch_mm(probe_sr, st, View.of(a), View.of(b), View.of(ref))
        got = torch.empty((128, 128), dtype=torch.int32, device=dev)
        from .mm import _copy2d_raw
        _copy2d_raw(dev, got, self.own_ptr, self.m * self.itemsize)
        torch.cuda.synchronize(dev)
        ok = ok and bool(torch.equal(got, ref))
        flags = [None] * self.world
        dist.all_gather_object(flags, ok, group=self.group)
        return all(flags)

    def _flags(self, j: int, owner: int) -> int:
        """Fold flags of launch j: remote or shared-with-a-peer folds at system scope."""
        nat = self.nat
        if owner != self.rank or self.shared[j]:
            return nat.MM_ATOMIC | (nat.MM_SYS if self.remote_bulk else nat.MM_REMOTE)
        return nat.MM_ATOMIC

    def _fill_owned(self, st, every: bool = False) -> None:
        """Semiring zero into the owned rectangles only (every fold, local or
        remote, lands inside them; the rest of the buffer is never read) --
        except those a sole-writer launch overwrites, unless ``every``."""
        from .mm import launch_fill

        mine = self.views[self.rank]
        for (i0, j0, n, m) in (self.owned if every else self.fill_rects):
            launch_fill(self.semiring.kernel_id, st, mine.sub(i0, j0, n, m))

    def _device_barrier(self) -> None:
        """Every rank's work enqueued so far is done before any rank's next work.

        NCCL: a one-element all-reduce, stream-ordered -- the host never
        blocks, the GPUs wait for each other (the collective completes only
        when every rank's stream reached it).  gloo (CPU tests, ranks sharing
        one GPU): synchronize + host barrier."""
        if self._nccl:
            dist.all_reduce(self._tok, group=self.group)
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)

    def run(self, A: torch.Tensor, B: torch.Tensor, C_init: torch.Tensor | None = None) -> None:
        from .device import View
        from .mm import launch_fill, launch_fold, launch_mm

        st = torch.cuda.current_stream(self.device)
        mine = self.views[self.rank]
        self._fill_owned(st)
        if C_init is not None:
            ci = View.of(C_init)
            for (i0, j0, n, m) in self.owned:
                if (i0, j0, n, m) not in self.fill_rects:   # a sole writer would overwrite it: fill first
                    launch_fill(self.semiring.kernel_id, st, mine.sub(i0, j0, n, m))
                launch_fold(self.semiring.kernel_id, st, mine.sub(i0, j0, n, m), ci.sub(i0, j0, n, m), False)
        if self.exchange:
            self._device_barrier()              # every owner's C is initialised
        av, bv = View.of(A), View.of(B)
        es = self.itemsize
        for j, ((ai, al, an, ak), (bl, bj, bk, bm), owner, (ci, cj, cn, cm)) in enumerate(self.launches):
            a, b = av.sub(ai, al, an, ak), bv.sub(bl, bj, bk, bm)
            if owner != self.rank and self.fold_style == "stage":
                t = self.temps[j]
                launch_mm(self.kid, st, a, b, View.of(t), overwrite=True, device=self.device)
                slot = self.stage_ptrs[owner] + self.outgoing[j] * es
                self.nat.check(self.nat.load().paco_copy2d(self.device, st.cuda_stream, slot, cm * es, t.data_ptr(),
                                                           t.stride(0) * es, cm * es, cn))
                continue
            if self.sole[j] and C_init is None:
                launch_mm(self.kid, st, a, b, mine.sub(ci, cj, cn, cm), overwrite=True, device=self.device)
                continue
            launch_mm(self.kid, st, a, b, self.views[owner].sub(ci, cj, cn, cm), flags=self._flags(j, owner),
                      device=self.device)
        if not self.exchange:
            return
        self._device_barrier()                  # every remote fold / staged block has landed
        for (ci, cj, cn, cm), off in self.incoming:
            src = View.raw(self.stage_ptr + off * es, cn, cm, es, self.device, ld=cm)
            launch_fold(self.semiring.kernel_id, st, mine.sub(ci, cj, cn, cm), src, False)
        # (a sender refills this rank's staging slots only after the next step's
        # first barrier, which this rank's stream reaches after these folds)

    def run_host(self, A_h: torch.Tensor, B_h: torch.Tensor, C_h: torch.Tensor) -> tuple[int, int]:
        """End to end from pinned host operands: C_h's owned rectangles <- C.

        Each rank uploads only the blocks of A and B its launches read, in k
        chunks of growing width on a copy stream (``mm._kphased_edges``), and
        folds each chunk into the owners' C as soon as it lands -- the atomic
        epilogue makes a k-chunked launch the same product, since C starts at
        the semiring zero.  After the barrier that makes every remote fold
        visible, the rank's owned rectangles of C are read back into ``C_h``
        (every rank holds the full-size host C, as every rank holds A_h, B_h
        in the reference's shared-memory setting).  Returns (H2D, D2H) bytes.
        """
        from .device import View
        from .mm import _PIPE_MIN_ROWS, _copy2d, _kphased_edges, launch_fill, launch_fold, launch_mm

        dev, es = self.device, self.itemsize
        st = torch.cuda.current_stream(dev)
        if getattr(self, "_host_bufs", None) is None or self._host_bufs[0].shape != A_h.shape \
                or self._host_bufs[1].shape != B_h.shape:
            self._host_bufs = (torch.empty(tuple(A_h.shape), dtype=A_h.dtype, device=dev),
                               torch.empty(tuple(B_h.shape), dtype=B_h.dtype, device=dev),
                               torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
        a_d, b_d, h2d, d2h = self._host_bufs
        # no exchange and disjoint launch rectangles: every C row block is final as
        # soon as this rank's last k chunk for it ran -- return it while the next
        # block computes (the row-blocked last phase of mm._kphased_host_mm)
        rects = [x[3] for x in self.launches]
        streamed = not self.exchange and all(_rect_intersect(r, q) is None
                                             for i, r in enumerate(rects) for q in rects[i + 1:])
        returned = []
        d2h.wait_stream(st)
        av, bv = View.of(a_d), View.of(b_d)
        mine = self.views[self.rank]
        self._fill_owned(st, every=True)        # k-chunked launches fold into C: all of it starts at zero
        if self.exchange:
            self._device_barrier()              # every owner's C is initialised
        h2d.wait_stream(st)
        sent_a, sent_b, h2d_bytes = set(), set(), 0
        for j, ((ai, al, an, ak), (bl, bj, bk, bm), owner, (ci, cj, cn, cm)) in enumerate(self.launches):
            staged = owner != self.rank and self.fold_style == "stage"
            if staged or ak < 256:
                spans = [(0, ak)]
            else:
                edges, front = _kphased_edges(ak)
                spans = list(zip(edges[:-1], edges[1:])) + [(front, ak)]
            for (l0, l1) in spans:
                ka = (ai, an, al + l0, al + l1)
                if ka not in sent_a:
                    sent_a.add(ka)
                    _copy2d(h2d, a_d, ai, al + l0, A_h, ai, al + l0, an, l1 - l0)
                    h2d_bytes += an * (l1 - l0) * es
                kb = (bj, bm, bl + l0, bl + l1)
                if kb not in sent_b:
                    sent_b.add(kb)
                    _copy2d(h2d, b_d, bl + l0, bj, B_h, bl + l0, bj, l1 - l0, bm)
                    h2d_bytes += bm * (l1 - l0) * es
                ev = torch.cuda.Event()
                ev.record(h2d)
                st.wait_event(ev)
                a, b = av.sub(ai, al + l0, an, l1 - l0), bv.sub(bl + l0, bj, l1 - l0, bm)
                if staged:
                    t = self.temps[j]
                    launch_mm(self.kid, st, a, b, View.of(t), overwrite=True, device=dev)
                    slot = self.stage_ptrs[owner] + self.outgoing[j] * es
                    self.nat.check(self.nat.load().paco_copy2d(dev, st.cuda_stream, slot, cm * es, t.data_ptr(),
                                                               t.stride(0) * es, cm * es, cn))
                    continue
                flags = self._flags(j, owner)
                if streamed and len(spans) > 1 and (l0, l1) == spans[-1] and an >= 2 * _PIPE_MIN_ROWS:
                    R = max(1, min(16, an // _PIPE_MIN_ROWS))
                    redges = [((an * i // R) // 128) * 128 for i in range(R)] + [an]
                    for r0, r1 in zip(redges[:-1], redges[1:]):
                        launch_mm(self.kid, st, av.sub(ai + r0, al + l0, r1 - r0, l1 - l0), b,
                                  self.views[owner].sub(ci + r0, cj, r1 - r0, cm), flags=flags, device=dev)
                        done = torch.cuda.Event()
                        done.record(st)
                        d2h.wait_event(done)
                        self.nat.check(self.nat.load().paco_copy2d(
                            dev, d2h.cuda_stream, C_h.data_ptr() + ((ci + r0) * C_h.stride(0) + cj) * es,
                            C_h.stride(0) * es, self.own_ptr + ((ci + r0) * self.m + cj) * es, self.m * es,
                            cm * es, r1 - r0))
                    returned.append((ci, cj, cn, cm))
                    continue
                launch_mm(self.kid, st, a, b, self.views[owner].sub(ci, cj, cn, cm), flags=flags, device=dev)
        if self.exchange:
            self._device_barrier()              # every remote fold / staged block has landed
        for (ci, cj, cn, cm), off in self.incoming:
            src = View.raw(self.stage_ptr + off * es, cn, cm, es, dev, ld=cm)
            launch_fold(self.semiring.kernel_id, st, mine.sub(ci, cj, cn, cm), src, False)
        d2h_bytes = sum(r[2] * r[3] * es for r in returned)
        for (i0, j0, n, m) in self.owned:
            for x in returned:  # rows already streamed back
                if _rect_intersect(x, (i0, j0, n, m)) == (i0, j0, n, m):
                    break
            else:
                self.nat.check(self.nat.load().paco_copy2d(
                    dev, st.cuda_stream, C_h.data_ptr() + (i0 * C_h.stride(0) + j0) * es, C_h.stride(0) * es,
                    self.own_ptr + (i0 * self.m + j0) * es, self.m * es, m * es, n))
                d2h_bytes += n * m * es
        st.wait_stream(d2h)
        torch.cuda.synchronize(dev)
        return h2d_bytes, d2h_bytes

    def gather(self, out: torch.Tensor, dst: int = 0) -> None:
        """Copy this rank's owned C rectangles into ``out`` (semiring zero
        elsewhere) and reduce the owners' pieces onto ``dst``."""
        from .device import View
        from .mm import launch_fill

        st = torch.cuda.current_stream(self.device)
        launch_fill(self.semiring.kernel_id, st, View.of(out))
        es = self.itemsize
        for (i0, j0, n, m) in self.owned:
            self.nat.check(self.nat.load().paco_copy2d(
                self.device, st.cuda_stream, out.data_ptr() + (i0 * out.stride(0) + j0) * es, out.stride(0) * es,
                self.own_ptr + (i0 * self.m + j0) * es, self.m * es, m * es, n))
        dist.reduce(out, dst=dst, op=self.op, group=self.group)

    def close(self) -> None:
        lib = self.nat.load()
        for r, p in enumerate(self.ptrs):
            if r != self.rank:
                lib.paco_ipc_close(self.device, p)
        for r, p in enumerate(self.stage_ptrs):
            if p is not None and r != self.rank:
                lib.paco_ipc_close(self.device, p)
        if self.stage_ptr is not None:
            lib.paco_device_free(self.device, self.stage_ptr)
        lib.paco_device_free(self.device, self.own_ptr)
        self.ptrs, self.stage_ptrs, self.stage_ptr = [], [None] * self.world, None


# ------------------------------------------------------------------ Strassen

class CudaStrassenOps:
    """Device arithmetic for ``DistributedStrassen`` (sm_100a kernels)."""

    def __init__(self, dtype: torch.dtype, stream: torch.cuda.Stream | None = None):
        from . import strassen as S

        self.S = S
        self.dtype = dtype
        self.kid, self.dt = S._RING[dtype]
        self.stream = stream

    def _st(self, t: torch.Tensor):
        return self.stream or torch.cuda.current_stream(t.device)

    def zeros(self, shape, like: torch.Tensor) -> torch.Tensor:
        return torch.zeros(shape, dtype=like.dtype, device=like.device)

    def lincomb(self, out: torch.Tensor, terms, accumulate: bool) -> None:
        from .device import View

        self.S._lincomb(self.dt, self._st(out), View.of(out), [(c, View.of(t)) for c, t in terms], accumulate)

    def strassen(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, base: int) -> None:
        from .device import View

        self.S._strassen_dev(View.of(a), View.of(b), View.of(out), base, self.dtype, self._st(out))

    def mm(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
        from .device import View
        from .mm import launch_mm

        launch_mm(self.kid, self._st(out), View.of(a), View.of(b), View.of(out), overwrite=True)

    def strassen_into(self, a: torch.Tensor, b: torch.Tensor, dests, base: int) -> bool:
        """dests = [(sign, C block)] (+/-)= a x b with the combinations folded into
        the leaf epilogues (fp32 only); False: not applicable here."""
        from .device import View

        if self.dtype != torch.float32:
            return False
        return self.S.strassen_into(View.of(a), View.of(b), [(View.of(d), sg) for sg, d in dests], base,
                                    self._st(a))


def strassen_placements(path: tuple[int, ...], size: int) -> list[tuple[int, int, int]]:
    """Where the product of tree node ``path`` lands in C: (sign, row, col) of
    each signed copy, the block being ``size >> len(path)`` square.

    Composes the C-block formulas top-down: at each level
    M_r is added with coefficient c into every quadrant whose formula holds r
    (M1 -> C00, C11; M2 -> C10, -C11; ...), inside the block its parent landed in.
    """
    from .strassen import C_TERMS

    out = [(1, 0, 0)]
    h = size
    for r in path:
        h //= 2
        nxt = []
        for s, i, j in out:
            for q, terms in C_TERMS.items():
                for c, rr in terms:
                    if rr == r:
                        nxt.append((s * c, i + int(q[0]) * h, j + int(q[1]) * h))
        out = nxt
    return out


class DistributedStrassen:
    """One process per GPU for a Strassen plan.

    A and B are replicated, so every rank forms the S/T operands of its own
    tree nodes locally (the path's S_r / T_r formulas applied level by level,
    shared prefixes formed once) and multiplies them (``strassen_seq`` of the
    node; for fp32 the single-GPU leaves: tf32 + 2 x bf16 products on raw
    operands when the node's leaf batch fills the CTA pairs, else 3xTF32).  Each product is added, with the signs of
    the C-block formulas composed along its path (``strassen_placements``),
    into a rank-local partial C; the pieces of split leftover leaves
    (``split_leftover``) are added the same way at their cuboid's final place
    inside the leaf product, so a k-cut pair's fold is part of the sum.  C is
    then ONE signed-sum reduce-scatter of the partials (NCCL): rank r holds
    rows [r*R, (r+1)*R) of C; ``gather`` assembles the whole C on one rank.
    The plan's FORM / COMBINE / REDUCE tasks need no execution of their own
    here: forming is per rank, combining and folding are the reduce-scatter.
    """

    def __init__(self, plan: Plan, ops, *, group=None):
        from .strassen import LeafPiece, StrassenNode

        meta = plan.meta
        if meta.get("algo") != "strassen":
            raise PlanError("not a Strassen plan")
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if plan.p != self.world:
            raise PlanError(f"plan built for p={plan.p}, world size is {self.world}")
        plan.validate()
        self.plan, self.ops, self.group = plan, ops, group
        self.n, self.size, self.base = meta["n"], meta["n_padded"], meta["base"]
        self.rows = -(-self.size // self.world)   # C rows per rank after the reduce-scatter
        self.nodes: list = []    # (path, StrassenNode)
        self.pieces: list = []   # (path, LeafPiece, (row, col) of the piece inside the leaf product)
        from .mm import fold_destinations
        dests = {}
        for t in plan.tasks:
            if t.kind != COMPUTE or t.worker != self.rank:
                continue
            if isinstance(t.region, LeafPiece):
                leaf = t.region.node
                mp = meta["split_leaves"][str(leaf)]
                if str(leaf) not in dests:
                    dests[str(leaf)] = fold_destinations(mp)
                cb = t.region.cuboid
                _, fi, fj = dests[str(leaf)].get(cb.out, (0, 0, 0))
                self.pieces.append((leaf.path, t.region, (fi + cb.out_i0, fj + cb.out_j0)))
            elif isinstance(t.region, StrassenNode):
                self.nodes.append((t.region.path, t.region))

    def _operands(self, A: torch.Tensor, B: torch.Tensor, path: tuple[int, ...], cache: dict):
        """S and T of tree node ``path``: the S_r / T_r formulas applied level by level."""
        from .strassen import S_TERMS, T_TERMS

        if path in cache:
            return cache[path]
        if not path:
            return A, B
        pa, pb = self._operands(A, B, path[:-1], cache)
        r = path[-1]
        h = pa.shape[0] // 2

        def quad(x, q):
            return x[int(q[0]) * h:(int(q[0]) + 1) * h, int(q[1]) * h:(int(q[1]) + 1) * h]

        res = []
        for src, terms in ((pa, S_TERMS[r]), (pb, T_TERMS[r])):
            if len(terms) == 1 and terms[0][0] == 1:
                res.append(quad(src, terms[0][1]))
                continue
            out = self.ops.zeros((h, h), src)
            self.ops.lincomb(out, [(c, quad(src, q)) for c, q in terms], False)
            res.append(out)
        cache[path] = tuple(res)
        return cache[path]

    def partial(self, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
        """This rank's signed partial C (rows padded to world * rows)."""
        N = self.size
        if tuple(A.shape) != (N, N) or tuple(B.shape) != (N, N):
            raise ValueError(f"operands must be padded to {N}x{N}, got A{tuple(A.shape)} B{tuple(B.shape)}")
        Cp = self.ops.zeros((self.rows * self.world, N), A)
        cache: dict = {}
        for path, nd in self.nodes:
            s, t = self._operands(A, B, path, cache)
            h = nd.size
            places = strassen_placements(path, N)
            into = getattr(self.ops, "strassen_into", None)
            if into is not None and into(s, t, [(sign, Cp[i:i + h, j:j + h]) for sign, i, j in places], self.base):
                continue  # the leaf epilogues folded every signed copy into Cp
            M = self.ops.zeros((h, h), A)
            self.ops.strassen(s, t, M, self.base)
            for sign, i, j in places:
                self.ops.lincomb(Cp[i:i + h, j:j + h], [(sign, M)], True)
        for path, piece, (ri, rj) in self.pieces:
            s, t = self._operands(A, B, path, cache)
            cb = piece.cuboid
            P = self.ops.zeros((cb.n, cb.m), A)
            self.ops.mm(s[cb.i0:cb.i0 + cb.n, cb.l0:cb.l0 + cb.k], t[cb.l0:cb.l0 + cb.k, cb.j0:cb.j0 + cb.m], P)
            for sign, i, j in strassen_placements(path, N):
                self.ops.lincomb(Cp[i + ri:i + ri + cb.n, j + rj:j + rj + cb.m], [(sign, P)], True)
        return Cp

    def run(self, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
        """Rows [rank*rows, (rank+1)*rows) of C = A x B (padded size; rows past
        the padded size are zero)."""
        Cp = self.partial(A, B)
        slab = self.ops.zeros((self.rows, self.size), A)
        _reduce_scatter_sum(slab, Cp, self.group)
        return slab

    def gather(self, slab: torch.Tensor, dst: int = 0) -> torch.Tensor | None:
        """The whole n x n C on ``dst`` (None elsewhere)."""
        full = self.ops.zeros((self.rows * self.world, self.size), slab)
        _all_gather(full, slab, self.group)
        return full[:self.n, :self.n] if self.rank == dst else None


def _gloo(group) -> bool:
    return dist.get_backend(group) == "gloo"


def _reduce_scatter_sum(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    """out = rank's row slab of the SUM of every rank's ``inp`` (NCCL
    reduce-scatter; gloo, which has none, does all-reduce + slice on host copies)."""
    if dist.get_world_size(group) == 1:
        out.copy_(inp)
        return
    if not _gloo(group):
        dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=group)
        return
    h = inp.cpu()
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    r, rows = dist.get_rank(group), out.shape[0]
    out.copy_(h[r * rows:(r + 1) * rows])


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    if dist.get_world_size(group) == 1:
        out.copy_(inp)
        return
    if not _gloo(group):
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    parts = [torch.empty_like(inp, device="cpu") for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, inp.cpu(), group=group)
    out.copy_(torch.cat(parts))

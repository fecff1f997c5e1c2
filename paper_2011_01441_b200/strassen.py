"""PACO-Strassen on B200 (the reference specifies it but ships no code).

Follows SPEC.md:474-552 and the identities of PAPER.md:1839-1852:

* ``strassen_seq(A, B, n, base=64)`` -- C = A x B with Strassen's 7-way
  recursion down to ``base`` (B_str), then classic semiring MM leaves
  (``mm_seq`` -> the sm_100a kernels; fp32 leaves as batched 3xTF32).  S_r/T_r
  formation and the C-block combination are ``paco_lincomb`` launches.
  Non-power-of-two n is zero-padded.
* ``strassen_paco_partition(n, p, base)`` -- pruned BFS of the arity-7 tree
  (core.py:149-222 with arity 7); every internal node gets a FORM task (its
  S/T additions, charged to the workers of its subtree, before its children)
  and a COMBINE task (its C-block additions, after all seven children).
* ``strassen_const_pieces_partition(n, p, cfg)`` -- the same, but after
  ``cfg.gamma`` super-rounds every still-unassigned node is dealt out
  round-robin (Corollary strassen-const-pieces).
* ``strassen_execute(plan, A, B)`` -- runs a plan on the GPU(s): workers map
  to (device, stream); returns C.

Ring: float32 (3xTF32 tcgen05 leaves), float64 (DFMA leaves) or int64 (exact).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .device import View, pick_device, stage_in
from .engine import execute_plan
from .mm import launch_fill, launch_fold, launch_mm
from .plan import COMPUTE, MERGE, REDUCE, Plan, PlanError, Task, pruned_bfs_assign

DEFAULT_STRASSEN_BASE = 64

# S_r, T_r and C-block formulas, 1-indexed as in PAPER.md:1839-1852:
# (coefficient, quadrant "rc") of A for S_r, of B for T_r; (coefficient, r) of M for C blocks.
S_TERMS = {1: ((1, "00"), (1, "11")), 2: ((1, "10"), (1, "11")), 3: ((1, "00"),), 4: ((1, "11"),),
           5: ((1, "00"), (1, "01")), 6: ((1, "10"), (-1, "00")), 7: ((1, "01"), (-1, "11"))}
T_TERMS = {1: ((1, "00"), (1, "11")), 2: ((1, "00"),), 3: ((1, "01"), (-1, "11")),
           4: ((1, "10"), (-1, "00")), 5: ((1, "11"),), 6: ((1, "00"), (1, "01")),
           7: ((1, "10"), (1, "11"))}
C_TERMS = {"00": ((1, 1), (1, 4), (-1, 5), (1, 7)), "01": ((1, 3), (1, 5)),
           "10": ((1, 2), (1, 4)), "11": ((1, 1), (1, 3), (-1, 2), (1, 6))}

# where M_r lands in C (the inverse of C_TERMS): r -> ((coef, quadrant), ...)
M_DESTS = {r: tuple((c, q) for q, terms in C_TERMS.items() for c, rr in terms if rr == r) for r in range(1, 8)}

_RING = {  # torch dtype -> (leaf kernel id, lincomb dtype id)
    torch.float32: (nat.SR_F32_TC, nat.DT_F32),   # 3xTF32 tensor-core leaves
    torch.float64: (nat.SR_F64, nat.DT_F64),
    torch.int64: (nat.SR_INT_I64, nat.DT_I64),
}


@dataclass(frozen=True)
class SuperRoundCfg:
    """Cap on assignment super-rounds for Strassen-Const-Pieces."""

    gamma: int = 8

    def __post_init__(self):
        if self.gamma < 1:
            raise PlanError(f"gamma must be >= 1, got {self.gamma}")


class StrassenNode:
    """One multiplication of the 7-way tree: ``path`` = sequence of r in 1..7."""

    __slots__ = ("path", "size", "kids", "task_id")

    def __init__(self, path: tuple[int, ...], size: int):
        self.path = path
        self.size = size
        self.kids: list[StrassenNode] = []
        self.task_id: int | None = None

    @property
    def depth(self) -> int:
        return len(self.path)

    @property
    def volume(self) -> int:
        """Strassen work of the node: 7^log2(size) (= size^log2 7) leaf-size units."""
        return 7 ** int(round(math.log2(self.size))) if self.size >= 1 else 0

    def __str__(self) -> str:
        return "strassen[depth=%d,path=%s,n=%d]" % (self.depth, ".".join(map(str, self.path)) or "-",
                                                   self.size)


@dataclass(frozen=True)
class LeafPiece:
    """One GPU's cuboid of a leftover leaf product M = S T, split across all p
    workers by MM-1-Piece.  ``cuboid`` is in the leaf's (i, j, l)
    space; its C face lands in M (out = 0) or in k-cut temporary ``out``."""

    node: StrassenNode
    cuboid: object

    def __str__(self) -> str:
        c = self.cuboid
        return f"piece[{self.node},i0={c.i0},j0={c.j0},l0={c.l0},n={c.n},m={c.m},k={c.k},out={c.out}]"


@dataclass(frozen=True)
class LeafFold:
    """k-cut REDUCE of a split leaf: (out, oi, oj) (+)= temp (matmul.py:455-460)."""

    node: StrassenNode
    temp: int
    out: int
    oi: int
    oj: int
    n: int
    m: int

    def __str__(self) -> str:
        return f"reduce[{self.node},temp={self.temp}->out={self.out},n={self.n},m={self.m}]"


def _padded(n: int) -> int:
    if n < 1:
        raise PlanError("n must be >= 1")
    return 1 << (n - 1).bit_length()


def _expand(node: StrassenNode) -> list[StrassenNode]:
    node.kids = [StrassenNode(node.path + (r,), node.size // 2) for r in range(1, 8)]
    return node.kids


def _assemble(root: StrassenNode, assigned: list[Task], p: int, n: int, base: int, variant: str,
              split: list | None = None) -> Plan:
    """Topological task list: FORM(internal, BFS) -> COMPUTE(assigned) -> COMBINE(reverse BFS).

    ``split``: (leaf, one-piece MM plan over p workers) pairs -- leaves computed
    as p cuboids plus their k-cut REDUCE tasks instead of by one worker."""
    internal: list[StrassenNode] = []
    frontier = [root]
    while frontier:
        nxt = []
        for nd in frontier:
            if nd.kids:
                internal.append(nd)
                nxt.extend(nd.kids)
        frontier = nxt
    owner = {id(t.region): t.worker for t in assigned}
    split = split or []
    everyone = tuple(range(p))

    workers_of: dict[int, tuple[int, ...]] = {id(leaf): everyone for leaf, _ in split}

    def subtree(nd: StrassenNode) -> tuple[int, ...]:
        key = id(nd)
        if key not in workers_of:
            if key in owner:
                workers_of[key] = (owner[key],)
            else:
                workers_of[key] = tuple(sorted({w for k in nd.kids for w in subtree(k)}))
        return workers_of[key]

    def pack(ws):
        return ws[0] if len(ws) == 1 else ws

    tasks: list[Task] = []
    form_id: dict[int, int] = {}
    parent_of: dict[int, StrassenNode] = {id(k): nd for nd in internal for k in nd.kids}
    for nd in internal:
        par = parent_of.get(id(nd))
        half = (nd.size // 2) ** 2
        t = Task(id=len(tasks), kind=MERGE, region=f"form[{nd}]", worker=pack(subtree(nd)),
                 deps=(form_id[id(par)],) if par is not None else (), cost_work=10 * half)
        form_id[id(nd)] = t.id
        tasks.append(t)
    done_id: dict[int, int] = {}
    for a in assigned:
        nd = a.region
        par = parent_of.get(id(nd))
        t = Task(id=len(tasks), kind=COMPUTE, region=nd, worker=a.worker,
                 deps=(form_id[id(par)],) if par is not None else (), cost_work=nd.volume, label=a.label)
        nd.task_id = t.id
        done_id[id(nd)] = (t.id,)
        tasks.append(t)
    label = max((a.label for a in assigned), default=0) + 1
    leaf_plans = {}
    for leaf, mplan in split:
        par = parent_of.get(id(leaf))
        pre = (form_id[id(par)],) if par is not None else ()
        vol = leaf.volume / float(leaf.size) ** 3  # Strassen work units per term
        new_id: dict[int, int] = {}
        for mt in mplan.tasks:
            if mt.kind == COMPUTE:
                region = LeafPiece(leaf, mt.region)
                kind, deps = COMPUTE, pre
                cost = max(1, round(vol * mt.region.n * mt.region.m * mt.region.k))
            else:
                spec = mplan.meta["reduces"][mt.id]
                region = LeafFold(leaf, *spec)
                kind, deps = REDUCE, tuple(new_id[d] for d in mt.deps)
                cost = max(1, round(vol * mt.cost_work))
            t = Task(id=len(tasks), kind=kind, region=region, worker=mt.worker, deps=deps,
                     cost_work=cost, label=label)
            new_id[mt.id] = t.id
            tasks.append(t)
        done_id[id(leaf)] = tuple(new_id.values())
        leaf_plans[str(leaf)] = mplan
    for nd in reversed(internal):
        half = (nd.size // 2) ** 2
        t = Task(id=len(tasks), kind=MERGE, region=f"combine[{nd}]", worker=pack(subtree(nd)),
                 deps=tuple(sorted(d for k in nd.kids for d in done_id[id(k)])), cost_work=8 * half)
        done_id[id(nd)] = (t.id,)
        tasks.append(t)
    temp = sum(21 * (nd.size // 2) ** 2 for nd in internal)
    temp += sum(sum(mp.meta["temp_sizes"].values()) for _, mp in split)
    meta = {"algo": "strassen", "variant": variant, "n": n, "n_padded": root.size, "base": base,
            "internal": len(internal), "leaves": len(assigned) + len(split), "temp_peak": temp,
            "tree": root, "split_leaves": leaf_plans}
    return Plan(tasks=tasks, p=p, meta=meta)


def strassen_paco_partition(n: int, p: int, base: int = DEFAULT_STRASSEN_BASE, *,
                            split_leftover: bool = False) -> Plan:
    """PACO-Strassen: pruned BFS of the 7-way tree.

    ``split_leftover`` (this build's extension): the final batch
    of fewer than p base-size leaves is not dealt one per worker -- which caps
    the efficiency at 49/56 = 87.5 % for p = 8, 49/54 = 90.7 % for p = 6 on
    cfg5 -- but each such leaf product is cut into p cuboids by MM-1-Piece
    (matmul.py:246-300) with its k-cut REDUCE tasks, so every worker gets an
    equal share."""
    from .cuboid import mm_one_piece_partition

    size = _padded(n)
    root = StrassenNode((), size)
    bfs = pruned_bfs_assign(root, 7, _expand, lambda nd: nd.size <= base, p,
                            cost=lambda nd: nd.volume)
    assigned, split = bfs.tasks, []
    if split_leftover and p > 1 and assigned:
        last = max(t.label for t in assigned)
        tail = [t for t in assigned if t.label == last]
        if len(tail) < p and all(t.region.size <= base and t.region.size ** 3 >= p for t in tail):
            assigned = [t for t in assigned if t.label != last]
            split = [(t.region, mm_one_piece_partition(t.region.size, t.region.size, t.region.size, p))
                     for t in tail]
    return _assemble(root, assigned, p, n, base, "paco+split-leftover" if split else "paco", split)


def strassen_const_pieces_partition(n: int, p: int, cfg: SuperRoundCfg = SuperRoundCfg(),
                                    base: int = DEFAULT_STRASSEN_BASE) -> Plan:
    """Strassen-Const-Pieces: pruned BFS capped at ``cfg.gamma`` super-rounds.

    A super-round ends when at least one batch fired at the current depth and
    fewer than p nodes survive; after the gamma-th, every
    surviving node is assigned round-robin in one final batch.
    """
    if p < 1:
        raise PlanError(f"need at least one worker, got p={p}")
    size = _padded(n)
    root = StrassenNode((), size)
    assigned: list[Task] = []
    cursor, label, rounds = 0, 0, 0

    def deal(nodes):
        nonlocal cursor, label
        label += 1
        for nd in nodes:
            assigned.append(Task(len(assigned), COMPUTE, nd, cursor, (), nd.volume, label))
            cursor = (cursor + 1) % p

    frontier = [root]
    while frontier:
        fired = False
        while len(frontier) >= p:
            deal(frontier[:p])
            frontier = frontier[p:]
            fired = True
        if not frontier:
            break
        if fired:
            rounds += 1
            if rounds >= cfg.gamma:
                deal(frontier)
                break
        if all(nd.size <= base for nd in frontier):
            deal(frontier)
            break
        nxt = []
        for nd in frontier:
            nxt.extend([nd] if nd.size <= base else _expand(nd))
        frontier = nxt
    return _assemble(root, assigned, p, n, base, f"const-pieces(gamma={cfg.gamma})")


# ---------------------------------------------------------------- device side

def _quad(v: View, q: str) -> View:
    h = v.rows // 2
    r, c = int(q[0]), int(q[1])
    return v.sub(r * h, c * h, h, h)


def _lincomb(dt: int, stream, out: View, terms, accumulate: bool = False) -> None:
    nin = len(terms)
    ins = (ctypes.c_void_p * nin)(*[t[1].ptr for t in terms])
    lds = (ctypes.c_int64 * nin)(*[t[1].ld for t in terms])
    coefs = (ctypes.c_int32 * nin)(*[t[0] for t in terms])
    nat.check(nat.load().paco_lincomb(out.device, stream.cuda_stream, dt, out.ptr, out.ld, out.rows,
                                      out.cols, nin, ins, lds, coefs, int(accumulate)))


def _single(terms) -> str | None:
    """The quadrant of a one-term, +1 formula (S3 = A00, T2 = B00, ...): used as a view."""
    return terms[0][1] if len(terms) == 1 and terms[0][0] == 1 else None


class _Workspace:
    """S/T/M buffers of one internal node: 7 of each, (size/2)^2, on one device.

    One-term formulas (S3, S4, T2, T5) are views of the operand quadrants,
    not copies.  ``leaf_split`` nodes (3xTF32 children) keep no S/T at all:
    their operands are formed straight into split tf32 pairs."""

    def __init__(self, size: int, dtype: torch.dtype, device: int, A: View, B: View, leaf_split: bool = False,
                 with_m: bool = True):
        h = size // 2

        def buf():
            return View.of(torch.empty((h, h), dtype=dtype, device=device))

        self.S = [None if leaf_split else (_quad(A, q) if (q := _single(S_TERMS[r])) else buf())
                  for r in range(1, 8)]
        self.T = [None if leaf_split else (_quad(B, q) if (q := _single(T_TERMS[r])) else buf())
                  for r in range(1, 8)]
        self.M = [buf() for _ in range(7)] if with_m else None


def _form(ws: _Workspace, A: View, B: View, dt: int, stream) -> None:
    for r in range(1, 8):
        if not _single(S_TERMS[r]):
            _lincomb(dt, stream, ws.S[r - 1], [(c, _quad(A, q)) for c, q in S_TERMS[r]])
        if not _single(T_TERMS[r]):
            _lincomb(dt, stream, ws.T[r - 1], [(c, _quad(B, q)) for c, q in T_TERMS[r]])


def _combine(ws: _Workspace, C: View, dt: int, stream) -> None:
    for q, terms in C_TERMS.items():
        _lincomb(dt, stream, _quad(C, q), [(c, ws.M[r - 1]) for c, r in terms])


def _split(stream, terms, src: View, hi: torch.Tensor, lo: torch.Tensor, transpose: bool) -> None:
    views = [_quad(src, q) for _, q in terms]
    nin = len(views)
    ins = (ctypes.c_void_p * nin)(*[v.ptr for v in views])
    lds = (ctypes.c_int64 * nin)(*[v.ld for v in views])
    coefs = (ctypes.c_int32 * nin)(*[c for c, _ in terms])
    h = views[0].rows
    nat.check(nat.load().paco_tf32_split(src.device, stream.cuda_stream, nin, ins, lds, coefs, h, h,
                                         int(transpose), hi.data_ptr(), lo.data_ptr(), hi.stride(0)))


def _leaf_level_tf32(A: View, B: View, C: View, stream) -> None:
    """A node whose seven children are 3xTF32 leaves: each S_r / T_r is formed
    directly as its split tf32 pair (A-side row-major, B-side transposed), so
    the sums never round-trip through HBM as fp32; then all seven products
    M_r = S_r T_r run as ONE batched tcgen05 launch (paco_mm_tf32x3, count 7:
    their tiles share one dynamic queue, so 7 x tiles fill the 148 SMs where
    one product's tiles alone quantise badly), and the C blocks are combined."""
    h = C.rows // 2
    ws = _Workspace(C.rows, torch.float32, C.device, A, B, leaf_split=True)
    ops = [[torch.empty((h, h), dtype=torch.float32, device=C.device) for _ in range(4)] for _ in range(7)]
    for r in range(1, 8):
        ah, al, bh, bl = ops[r - 1]
        _split(stream, S_TERMS[r], A, ah, al, transpose=False)
        _split(stream, T_TERMS[r], B, bh, bl, transpose=True)

    def arr(vals):
        return (ctypes.c_void_p * 7)(*vals)

    nat.check(nat.load().paco_mm_tf32x3(
        C.device, stream.cuda_stream, 7, arr([o[0].data_ptr() for o in ops]), arr([o[1].data_ptr() for o in ops]), h,
        arr([o[2].data_ptr() for o in ops]), arr([o[3].data_ptr() for o in ops]), h,
        arr([M.ptr for M in ws.M]), ws.M[0].ld, h, h, h, nat.MM_OVERWRITE))
    for o in ops:
        for t in o:
            t.record_stream(stream)
    _combine(ws, C, nat.DT_F32, stream)


def _leaf_level(n: int, base: int) -> bool:
    """A node of size n whose seven children are 3xTF32 leaves."""
    h = n // 2
    return n % 2 == 0 and (h <= base or h % 2) and h % 4 == 0


def _leaf_level_multi(A: View, B: View, dests, stream) -> None:
    """Leaf-level node whose product lands in ``dests`` [(View, sign)]: each
    child M_r = S_r T_r is folded by the GEMM epilogue straight into every C
    block it contributes to -- M_DESTS[r] inside each destination, signs
    multiplied (<= 4 blocks) -- so no M buffer is written and no combination
    pass reads one (paco_mm_tf32x3_multi, TMA reduce-adds)."""
    h = A.rows // 2
    dev = A.device
    if TF32B2 and _pair_batch(h, h, 7) and h % 8 == 0:
        _leaf_level_b2(A, B, dests, stream)
        return
    fuse_a = FUSED_A and _pair_batch(h, h, 7) and A.ptr % 16 == 0 and (A.ld * 4) % 16 == 0
    ops = [[torch.empty((h, h), dtype=torch.float32, device=dev) for _ in range(2 if fuse_a else 4)]
           for _ in range(7)]
    for r in range(1, 8):
        if fuse_a:
            bh, bl = ops[r - 1]
        else:
            ah, al, bh, bl = ops[r - 1]
            _split(stream, S_TERMS[r], A, ah, al, transpose=False)
        _split(stream, T_TERMS[r], B, bh, bl, transpose=True)
    ndst = (ctypes.c_int32 * 7)()
    dst = (ctypes.c_void_p * 28)()
    sign = (ctypes.c_int32 * 28)()
    ld = None
    for r in range(1, 8):
        targets = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
        if len(targets) > 4:
            raise ValueError("a leaf product folds into at most 4 C blocks")
        ndst[r - 1] = len(targets)
        for d, (v, sg) in enumerate(targets):
            dst[4 * (r - 1) + d] = v.ptr
            sign[4 * (r - 1) + d] = sg
            if ld is None:
                ld = v.ld
            elif v.ld != ld:
                raise ValueError("destinations must share one row pitch")

    def arr(vals):
        return (ctypes.c_void_p * 7)(*vals)

    if fuse_a:
        # S_r formed inside the pair kernel from A's quadrants (no A-side split launches)
        nta = (ctypes.c_int32 * 7)()
        at, asg = (ctypes.c_void_p * 14)(), (ctypes.c_int32 * 14)()
        for r in range(1, 8):
            nta[r - 1] = len(S_TERMS[r])
            for t, (c, q) in enumerate(S_TERMS[r]):
                at[2 * (r - 1) + t], asg[2 * (r - 1) + t] = _quad(A, q).ptr, c
        nat.check(nat.load().paco_mm_tf32x3_fused_a(
            dev, stream.cuda_stream, 7, nta, at, asg, A.ld, arr([o[0].data_ptr() for o in ops]),
            arr([o[1].data_ptr() for o in ops]), h, ndst, dst, sign, ld, h, h, h))
    else:
        nat.check(nat.load().paco_mm_tf32x3_multi(
            dev, stream.cuda_stream, 7, arr([o[0].data_ptr() for o in ops]), arr([o[1].data_ptr() for o in ops]), h,
            arr([o[2].data_ptr() for o in ops]), arr([o[3].data_ptr() for o in ops]), h, ndst, dst, sign, ld, h, h, h))
    for o in ops:
        for t in o:
            t.record_stream(stream)


def _leaf_level_b2(A: View, B: View, dests, stream) -> None:
    """The leaf level in the tf32 + 2 x bf16 format on CTA pairs: every S_r / T_r
    formed straight into (tf32 hi, bf16 hi, bf16 lo) -- T_r transposed --
    (``paco_tf32b2_split``), the seven products one ``paco_mm_tf32b2_multi``
    launch: hi*hi on the tf32 path, the two correction products as bf16 MMAs
    (half the tensor time), each folded (+/-) into its C blocks."""
    h = A.rows // 2
    dev = A.device
    lib = nat.load()
    cv = TF32B2_CONVERT   # bf16(hi) formed inside the kernel: 6 B of operand traffic per element, not 8
    bufs = []
    for r in range(1, 8):
        row = []
        for terms, src, tr in ((S_TERMS[r], A, False), (T_TERMS[r], B, True)):
            hi = torch.empty((h, h), dtype=torch.float32, device=dev)
            h16 = None if cv else torch.empty((h, h), dtype=torch.bfloat16, device=dev)
            l16 = torch.empty((h, h), dtype=torch.bfloat16, device=dev)
            views = [_quad(src, q) for _, q in terms]
            nin = len(views)
            nat.check(lib.paco_tf32b2_split(
                dev, stream.cuda_stream, nin, (ctypes.c_void_p * nin)(*[v.ptr for v in views]),
                (ctypes.c_int64 * nin)(*[v.ld for v in views]), (ctypes.c_int32 * nin)(*[c for c, _ in terms]),
                h, h, int(tr), hi.data_ptr(), None if cv else h16.data_ptr(), l16.data_ptr(), h))
            row += [hi, h16, l16]
        bufs.append(row)
    ndst = (ctypes.c_int32 * 7)()
    dst = (ctypes.c_void_p * 28)()
    sign = (ctypes.c_int32 * 28)()
    ld = None
    for r in range(1, 8):
        targets = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
        if len(targets) > 4:
            raise ValueError("a leaf product folds into at most 4 C blocks")
        ndst[r - 1] = len(targets)
        for d, (v, sg) in enumerate(targets):
            dst[4 * (r - 1) + d], sign[4 * (r - 1) + d] = v.ptr, sg
            if ld is None:
                ld = v.ld
            elif v.ld != ld:
                raise ValueError("destinations must share one row pitch")

    def arr(i):
        if row_none(i):
            return None
        return (ctypes.c_void_p * 7)(*[row[i].data_ptr() for row in bufs])

    def row_none(i):
        return bufs[0][i] is None

    nat.check(lib.paco_mm_tf32b2_multi(dev, stream.cuda_stream, 7, arr(0), arr(1), arr(2), h, arr(3), arr(4), arr(5), h,
                                       ndst, dst, sign, ld, h, h, h))
    for row in bufs:
        for t in row:
            if t is not None:
                t.record_stream(stream)


def _strassen_tc_fused(A: View, B: View, dests, base: int, stream) -> None:
    """dests (+/-)= A x B for the fp32 (3xTF32) ring, depth-first, with the
    C-block combinations folded into the leaf GEMMs' epilogues: a node hands
    each child the C blocks its M_r lands in (M_DESTS) instead of an M buffer,
    as long as the leaves then fold into <= 4 blocks; deeper trees materialise
    an M_r (zero-filled) at the level where that bound would break."""
    n = A.rows
    if _leaf_level(n, base) and len(dests) <= 2:
        _leaf_level_multi(A, B, dests, stream)
        return
    h = n // 2
    ws = _Workspace(n, torch.float32, A.device, A, B, with_m=False)
    _form(ws, A, B, nat.DT_F32, stream)
    for r in range(1, 8):
        child = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
        fits = len(child) <= (2 if _leaf_level(h, base) else 1)
        if h > base and h % 2 == 0 and fits:
            _strassen_tc_fused(ws.S[r - 1], ws.T[r - 1], child, base, stream)
            continue
        M = View.of(torch.empty((h, h), dtype=torch.float32, device=A.device))
        _strassen_dev(ws.S[r - 1], ws.T[r - 1], M, base, torch.float32, stream)
        for D, sd in child:
            _lincomb(nat.DT_F32, stream, D, [(sd, M)], accumulate=True)


def _tquad(q: str) -> str:
    """Quadrant (r, c) of B is quadrant (c, r) of B^T."""
    return q[1] + q[0]


def _transpose(src: View, stream) -> View:
    """A fresh row-major src^T (paco_transpose)."""
    out = View.of(torch.empty((src.cols, src.rows), dtype=torch.float32, device=src.device))
    nat.check(nat.load().paco_transpose(src.device, stream.cuda_stream, 4, out.ptr, out.ld, src.ptr, src.ld, src.rows,
                                        src.cols))
    out.tensor.record_stream(stream)
    return out


def _leaf_level_fused(A: View, Bt: View, dests, stream) -> None:
    """Leaf-level node, B given transposed: its seven products M_r = S_r T_r as
    ONE paco_mm_tf32x3_fused launch.  S_r's terms are A's quadrants, T_r^T's
    are B^T's (transposed quadrant names); the kernel forms each operand tile
    and splits it into tf32 hi/lo in shared memory, and the epilogue folds M_r
    (+/-) into every C block it lands in -- no split launches, no hi/lo or M
    buffers in HBM."""
    h = A.rows // 2
    nta, ntb = (ctypes.c_int32 * 7)(), (ctypes.c_int32 * 7)()
    at, bt = (ctypes.c_void_p * 14)(), (ctypes.c_void_p * 14)()
    asg, bsg = (ctypes.c_int32 * 14)(), (ctypes.c_int32 * 14)()
    ndst, dst, sign = (ctypes.c_int32 * 7)(), (ctypes.c_void_p * 28)(), (ctypes.c_int32 * 28)()
    ld = None
    for r in range(1, 8):
        q = r - 1
        nta[q], ntb[q] = len(S_TERMS[r]), len(T_TERMS[r])
        for t, (c, qq) in enumerate(S_TERMS[r]):
            at[2 * q + t], asg[2 * q + t] = _quad(A, qq).ptr, c
        for t, (c, qq) in enumerate(T_TERMS[r]):
            bt[2 * q + t], bsg[2 * q + t] = _quad(Bt, _tquad(qq)).ptr, c
        targets = [(_quad(D, qq), sd * c) for D, sd in dests for c, qq in M_DESTS[r]]
        if len(targets) > 4:
            raise ValueError("a leaf product folds into at most 4 C blocks")
        ndst[q] = len(targets)
        for d, (v, sg) in enumerate(targets):
            dst[4 * q + d], sign[4 * q + d] = v.ptr, sg
            if ld is None:
                ld = v.ld
            elif v.ld != ld:
                raise ValueError("destinations must share one row pitch")
    nat.check(nat.load().paco_mm_tf32x3_fused(A.device, stream.cuda_stream, 7, nta, at, asg, A.ld, ntb, bt, bsg, Bt.ld,
                                              ndst, dst, sign, ld, h, h, h))


def _form_all(src: View, table, transpose: bool, stream, keep: list, pitch: int | None = None) -> list:
    """The seven S_r (table = S_TERMS, from A) or T_r^T (T_TERMS, from B^T with
    transposed quadrant names) of a node: one-term formulas as quadrant views,
    every multi-term one written by ONE ``paco_lincomb_multi`` pass over the four
    quadrants (each read once).  New buffers get row pitch ``pitch`` (default h)."""
    h = src.rows // 2
    names = ("00", "01", "10", "11")
    quads = [_quad(src, _tquad(q) if transpose else q) for q in names]
    out, multi = [None] * 7, []
    for r in range(1, 8):
        terms = table[r]
        if len(terms) == 1 and terms[0][0] == 1:
            out[r - 1] = quads[names.index(terms[0][1])]
            continue
        buf = torch.empty((h, pitch or h), dtype=torch.float32, device=src.device)
        keep.append(buf)
        out[r - 1] = View.of(buf).sub(0, 0, h, h)
        row = [0] * 4
        for c, q in terms:
            row[names.index(q)] = c
        multi.append((out[r - 1], row))
    if multi:
        nat.check(nat.load().paco_lincomb_multi(
            src.device, stream.cuda_stream, h, h, 4, (ctypes.c_void_p * 4)(*[v.ptr for v in quads]),
            (ctypes.c_int64 * 4)(*[v.ld for v in quads]), len(multi),
            (ctypes.c_void_p * len(multi))(*[v.ptr for v, _ in multi]),
            (ctypes.c_int64 * len(multi))(*[v.ld for v, _ in multi]),
            (ctypes.c_int32 * (4 * len(multi)))(*[c for _, row in multi for c in row])))
    return out


def _leaf_level_b2raw(A: View, Bt: View, dests, stream) -> None:
    """Leaf-level node, B given transposed, leaves in the tf32 + 2 x bf16 format
    with NO split pass: each S_r (from A's quadrants) and T_r^T (from B^T's) is
    a quadrant view when it has one term, else one fp32 lincomb; the seven
    products are one ``paco_mm_tf32b2_multi`` launch on plain fp32 operands --
    the tf32 MMA reads x itself (hi = its top 19 bits) and the kernel forms
    bf16(hi) and bf16(x - hi) in shared memory (4 bytes of L2 traffic per
    element)."""
    h = A.rows // 2
    dev = A.device
    keep = []
    # sums take the node's row pitch, so views and sums share one operand pitch
    S_ = _form_all(A, S_TERMS, False, stream, keep, pitch=A.ld)
    T_ = _form_all(Bt, T_TERMS, True, stream, keep, pitch=Bt.ld)
    ops = list(zip(S_, T_))
    lda = {v.ld for v, _ in ops}
    ldb = {v.ld for _, v in ops}
    if len(lda) != 1 or len(ldb) != 1:
        raise ValueError("leaf operands must share one row pitch")
    ndst = (ctypes.c_int32 * 7)()
    dst = (ctypes.c_void_p * 28)()
    sign = (ctypes.c_int32 * 28)()
    ld = None
    for r in range(1, 8):
        targets = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
        if len(targets) > 4:
            raise ValueError("a leaf product folds into at most 4 C blocks")
        ndst[r - 1] = len(targets)
        for d, (v, sg) in enumerate(targets):
            dst[4 * (r - 1) + d], sign[4 * (r - 1) + d] = v.ptr, sg
            if ld is None:
                ld = v.ld
            elif v.ld != ld:
                raise ValueError("destinations must share one row pitch")
    arr = lambda vs: (ctypes.c_void_p * 7)(*[v.ptr for v in vs])  # noqa: E731
    nat.check(nat.load().paco_mm_tf32b2_multi(dev, stream.cuda_stream, 7, arr([a for a, _ in ops]), None, None,
                                              lda.pop(), arr([b for _, b in ops]), None, None, ldb.pop(), ndst, dst,
                                              sign, ld, h, h, h))
    for t in keep:
        t.record_stream(stream)


def _split_terms(terms, table, transpose: bool, stream, keep: list) -> list:
    """The seven S_r (table = S_TERMS) or T_r^T (T_TERMS, transposed quadrant
    names) of a leaf-level node whose operand is the signed sum of ``terms``
    [(coef, View)] (one view, or up to two level-0 blocks: the operand's
    quadrant q is then the sum of the terms' quadrants q, so the level-1 fp32
    sum is never materialised), as bf16x3 (hi, lo) plane pairs, all written by
    ONE ``paco_lincomb_split`` pass over the terms' quadrants (one-term formulas
    are split copies).  Returns [(hi, lo)] addresses of pitch h."""
    h = terms[0][1].rows // 2
    names = ("00", "01", "10", "11")
    ins = [_quad(v, _tquad(q) if transpose else q) for _, v in terms for q in names]
    planes = torch.empty((2, 7, h, h), dtype=torch.bfloat16, device=terms[0][1].device)
    keep.append(planes)
    coefs = []
    for r in range(1, 8):
        row = [0] * len(ins)
        for t, (c, _) in enumerate(terms):
            for c2, q in table[r]:
                row[4 * t + names.index(q)] = c * c2
        coefs += row
    his = [planes[0, r].data_ptr() for r in range(7)]
    los = [planes[1, r].data_ptr() for r in range(7)]
    ni = len(ins)
    nat.check(nat.load().paco_lincomb_split(
        terms[0][1].device, stream.cuda_stream, h, h, ni, (ctypes.c_void_p * ni)(*[v.ptr for v in ins]),
        (ctypes.c_int64 * ni)(*[v.ld for v in ins]), 7, (ctypes.c_void_p * 7)(*his), (ctypes.c_void_p * 7)(*los),
        (ctypes.c_int64 * 7)(*([h] * 7)), (ctypes.c_int32 * (7 * ni))(*coefs)))
    return list(zip(his, los))


def _split_all(src: View, table, transpose: bool, stream, keep: list) -> list:
    """``_split_terms`` of a node whose operand is the single view ``src``."""
    return _split_terms([(1, src)], table, transpose, stream, keep)


def _leaf_level_b3(A: View, Bt: View, dests, stream, pre=None, h: int | None = None, dev: int | None = None,
                   bnat: bool = False) -> None:
    """Leaf-level node, leaves in the bf16x3 format: the seven S_r and T_r^T (or,
    with ``bnat``, T_r in B's own k x m layout) are written as bf16 (hi, lo)
    planes by one ``paco_lincomb_split`` pass per side -- or arrive formed
    already as ``pre`` = (S planes, T planes, buffers to keep alive), with ``h``
    and ``dev`` -- and the seven products are one ``paco_mm_bf16x3_multi(_bn)``
    launch (hi*hi + hi*lo + lo*hi on kind::f16, fp32 accumulation) whose
    epilogues reduce-add each product with its signs into its C blocks
    (M_DESTS)."""
    if A is not None:
        h, dev = A.rows // 2, A.device
    if pre is None:
        keep = []
        S_ = _split_all(A, S_TERMS, False, stream, keep)
        T_ = _split_all(Bt, T_TERMS, not bnat, stream, keep)   # bnat: Bt is B itself (k x m)
    else:  # formed already from the level-0 blocks (_strassen_tc_fused_t, _strassen_b3n)
        S_, T_, keep = pre
    ndst = (ctypes.c_int32 * 7)()
    dst = (ctypes.c_void_p * 28)()
    sign = (ctypes.c_int32 * 28)()
    ld = None
    for r in range(1, 8):
        targets = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
        if len(targets) > 4:
            raise ValueError("a leaf product folds into at most 4 C blocks")
        ndst[r - 1] = len(targets)
        for d, (v, sg) in enumerate(targets):
            dst[4 * (r - 1) + d], sign[4 * (r - 1) + d] = v.ptr, sg
            if ld is None:
                ld = v.ld
            elif v.ld != ld:
                raise ValueError("destinations must share one row pitch")
    arr = lambda vs: (ctypes.c_void_p * 7)(*vs)  # noqa: E731
    fn = nat.load().paco_mm_bf16x3_multi_bn if bnat else nat.load().paco_mm_bf16x3_multi
    nat.check(fn(dev, stream.cuda_stream, 7, arr([a for a, _ in S_]), arr([a for _, a in S_]), h,
                 arr([b for b, _ in T_]), arr([b for _, b in T_]), h, ndst, dst, sign, ld, h, h, h))
    for t in keep:
        t.record_stream(stream)


def _default_leaf(n: int, base: int):
    """The leaf-level routine of the single-GPU fp32 Strassen path (B transposed
    once): bf16x3 (LEAF_BF16X3, leaf blocks a multiple of 8) or the raw-operand
    tf32 + 2 x bf16 format."""
    while n > base and n % 2 == 0:
        if _leaf_level(n, base):
            return _leaf_level_b3 if LEAF_BF16X3 and (n // 2) % 8 == 0 else _leaf_level_b2raw
        n //= 2
    return _leaf_level_b2raw


def _b3n_ok(n: int, base: int, dests) -> bool:
    """The bf16x3 leaves can take B in its own layout (no transpose): the node is a
    leaf-level node, or its children are (direct formation from its quadrants)."""
    if not (LEAF_BF16X3 and B3_NATURAL and B3_DIRECT) or n % 2:
        return False
    h = n // 2
    if _leaf_level(n, base):
        return h % 8 == 0 and len(dests) <= 2
    if not (_leaf_level(h, base) and h % 2 == 0 and (h // 2) % 8 == 0):
        return False
    return all(len([1 for _ in dests for _c in M_DESTS[r]]) <= 2 for r in range(1, 8))


def _strassen_b3n(A: View, B: View, dests, base: int, stream) -> None:
    """dests (+/-)= A x B in bf16x3 with B in its own k x m layout (``_b3n_ok``):
    T_r planes formed from B's quadrants and read by the MMA as MN-major tiles,
    so B is never transposed."""
    n = A.rows
    if _leaf_level(n, base):
        _leaf_level_b3(A, B, dests, stream, bnat=True)
        return
    h = n // 2
    hq = h // 2
    if B3_ONEPASS and n % 4 == 0 and hq % 8 == 0:
        # all 49 leaf operands of each side in one pass over the operand
        planes = torch.empty((2, 2, 49, hq, hq), dtype=torch.bfloat16, device=A.device)
        lib = nat.load()
        for side, X in ((0, A), (1, B)):
            his = (ctypes.c_void_p * 49)(*[planes[side, 0, o].data_ptr() for o in range(49)])
            los = (ctypes.c_void_p * 49)(*[planes[side, 1, o].data_ptr() for o in range(49)])
            nat.check(lib.paco_strassen_split49(A.device, stream.cuda_stream, side, X.ptr, X.ld, hq, his, los, hq))
        addr = lambda side, part, o: planes[side, part, o].data_ptr()  # noqa: E731
        for r in range(1, 8):
            child = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
            os_ = [7 * (r - 1) + r2 for r2 in range(7)]
            S_ = [(addr(0, 0, o), addr(0, 1, o)) for o in os_]
            T_ = [(addr(1, 0, o), addr(1, 1, o)) for o in os_]
            _leaf_level_b3(None, None, child, stream, pre=(S_, T_, []), h=hq, dev=A.device, bnat=True)
        planes.record_stream(stream)
        return
    for r in range(1, 8):
        child = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
        ck = []
        S_ = _split_terms([(c, _quad(A, q)) for c, q in S_TERMS[r]], S_TERMS, False, stream, ck)
        T_ = _split_terms([(c, _quad(B, q)) for c, q in T_TERMS[r]], T_TERMS, False, stream, ck)
        _leaf_level_b3(None, None, child, stream, pre=(S_, T_, ck), h=hq, dev=A.device, bnat=True)


def _strassen_tc_fused_t(A: View, Bt: View, dests, base: int, stream, leaf=None) -> None:
    """dests (+/-)= A x B for the fp32 (3xTF32) ring with B given as B^T (the
    fused-producer path): S_r from A's quadrants and T_r^T from B^T's, formed
    by lincomb above the leaf level only; at the leaf level the formation runs
    inside the GEMM (``_leaf_level_fused``).  C combinations fold into the leaf
    epilogues as in ``_strassen_tc_fused``."""
    n = A.rows
    if _leaf_level(n, base) and len(dests) <= 2:
        (leaf or _leaf_level_fused)(A, Bt, dests, stream)
        return
    h = n // 2
    dev = A.device
    keep = []
    kids = {r: [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]] for r in range(1, 8)}
    if (leaf is _leaf_level_b3 and B3_DIRECT and _leaf_level(h, base) and h % 2 == 0 and (h // 2) % 8 == 0
            and all(len(c) <= 2 for c in kids.values())):
        # leaf-level children: form each child's bf16x3 operands straight from this
        # node's quadrants (no level-1 fp32 sums), then its seven products
        for r in range(1, 8):
            child = kids[r]
            ck = []
            S_ = _split_terms([(c, _quad(A, q)) for c, q in S_TERMS[r]], S_TERMS, False, stream, ck)
            T_ = _split_terms([(c, _quad(Bt, _tquad(q))) for c, q in T_TERMS[r]], T_TERMS, True, stream, ck)
            _leaf_level_b3(None, None, child, stream, pre=(S_, T_, ck), h=h // 2, dev=dev)
        return
    S_all = _form_all(A, S_TERMS, False, stream, keep)
    T_all = _form_all(Bt, T_TERMS, True, stream, keep)
    children = {}
    for r in range(1, 8):
        child = [(_quad(D, q), sd * c) for D, sd in dests for c, q in M_DESTS[r]]
        fits = len(child) <= (2 if _leaf_level(h, base) else 1)
        children[r] = (child, h > base and h % 2 == 0 and fits)
    for r in range(1, 8):
        S, Tt = S_all[r - 1], T_all[r - 1]
        child, down = children[r]
        if down:
            _strassen_tc_fused_t(S, Tt, child, base, stream, leaf)
            continue
        M = View.of(torch.empty((h, h), dtype=torch.float32, device=dev))
        _strassen_dev(S, _transpose(Tt, stream), M, base, torch.float32, stream)
        for D, sd in child:
            _lincomb(nat.DT_F32, stream, D, [(sd, M)], accumulate=True)


def _b2raw_ok(n: int, base: int) -> bool:
    """The raw-operand tf32 + 2 x bf16 leaves apply: a halving chain to a leaf
    level whose seven products are a CTA-pair batch with 16-byte aligned views."""
    while n > base and n % 2 == 0:
        if _leaf_level(n, base):
            h = n // 2
            return h % 8 == 0 and _pair_batch(h, h, 7)
        n //= 2
    return False


def _fused_producer_ok(n: int, base: int) -> bool:
    """The fused-formation leaves apply: a square power-of-two-halving chain down
    to a leaf level whose blocks keep 16-byte aligned quadrant views."""
    while n > base and n % 2 == 0:
        if _leaf_level(n, base):
            return (n // 2) % 4 == 0
        n //= 2
    return False


def _leaf_multi(A: View, B: View, dests, stream) -> None:
    """One leaf product folded (+/-) into <= 4 blocks (count-1 batch): on CTA
    pairs in the raw-operand tf32 + 2 x bf16 format when it fills them (B
    transposed once), else 3xTF32 from split operands."""
    n, k = A.rows, A.cols
    m = B.cols
    dev = A.device
    if (TF32B2 and TF32B2_RAW and _pair_batch(n, m, 1) and A.ptr % 16 == 0 and A.ld % 4 == 0 and k % 4 == 0
            and all(d.ld == dests[0][0].ld for d, _ in dests)):
        Bt = _transpose(B, stream)
        one_v = lambda v: (ctypes.c_void_p * 1)(v.ptr)  # noqa: E731
        ndst = (ctypes.c_int32 * 1)(len(dests))
        dst = (ctypes.c_void_p * 4)(*[d.ptr for d, _ in dests])
        sign = (ctypes.c_int32 * 4)(*[sg for _, sg in dests])
        nat.check(nat.load().paco_mm_tf32b2_multi(dev, stream.cuda_stream, 1, one_v(A), None, None, A.ld, one_v(Bt),
                                                  None, None, Bt.ld, ndst, dst, sign, dests[0][0].ld, n, m, k))
        return
    kp = (k + 3) // 4 * 4
    ah = torch.empty((n, kp), dtype=torch.float32, device=dev)
    al = torch.empty_like(ah)
    bh = torch.empty((m, kp), dtype=torch.float32, device=dev)
    bl = torch.empty_like(bh)
    lib = nat.load()
    one = (ctypes.c_int32 * 1)(1)
    for src, rows, cols, tr, hi, lo in ((A, n, k, 0, ah, al), (B, k, m, 1, bh, bl)):
        nat.check(lib.paco_tf32_split(dev, stream.cuda_stream, 1, (ctypes.c_void_p * 1)(src.ptr),
                                      (ctypes.c_int64 * 1)(src.ld), one, rows, cols, tr, hi.data_ptr(),
                                      lo.data_ptr(), kp))
    ndst = (ctypes.c_int32 * 1)(len(dests))
    dst = (ctypes.c_void_p * 4)(*[d.ptr for d, _ in dests])
    sign = (ctypes.c_int32 * 4)(*[sg for _, sg in dests])
    one_p = lambda t: (ctypes.c_void_p * 1)(t.data_ptr())  # noqa: E731
    nat.check(lib.paco_mm_tf32x3_multi(dev, stream.cuda_stream, 1, one_p(ah), one_p(al), kp, one_p(bh), one_p(bl),
                                       kp, ndst, dst, sign, dests[0][0].ld, n, m, k))
    for t in (ah, al, bh, bl):
        t.record_stream(stream)


def strassen_into(A: View, B: View, dests, base: int, stream) -> bool:
    """dests (+/-)= A x B for fp32 operands with every C-block combination folded
    into the leaf epilogues (the executor of ``distributed.DistributedStrassen``
    hands a node its signed C placements).  Returns False when the fused path
    does not apply (alignment, more than 4 leaf destinations), so the caller
    takes the M-buffer path."""
    n = A.rows
    ok = FUSED_COMBINE and all(d.ptr % 16 == 0 and d.ld % 4 == 0 for d, _ in dests) and n % 4 == 0
    if not ok:
        return False
    if n <= base or n % 2:
        if len(dests) > 4:
            return False
        _leaf_multi(A, B, dests, stream)
        return True
    if A.ptr % 16 == 0 and A.ld % 4 == 0 and B.ptr % 16 == 0 and B.ld % 4 == 0 and _b3n_ok(n, base, dests):
        _strassen_b3n(A, B, dests, base, stream)   # the default: bf16x3, B in its own layout
        return True
    if TF32B2 and TF32B2_RAW and A.ptr % 16 == 0 and A.ld % 4 == 0 and _b2raw_ok(n, base):
        # the single-GPU leaves: plain fp32 operands, B transposed once
        _strassen_tc_fused_t(A, _transpose(B, stream), dests, base, stream, leaf=_default_leaf(n, base))
        return True
    if _leaf_level(n, base) and len(dests) > 2:
        return False
    _strassen_tc_fused(A, B, dests, base, stream)
    return True


# fp32 Strassen: fold the C-block combination into the leaf epilogues (True, the
# measured default) or materialise M buffers + lincomb (False; kept for A/B runs)
FUSED_COMBINE = True
# Form the leaf operands inside the 3xTF32 GEMM from B^T quadrants
# (paco_mm_tf32x3_fused) instead of split launches.  Off: measured slower on
# cfg5 (44 vs 34 ms) -- the in-smem formation adds ~89 KB
# of shared-memory traffic per 16-deep k block to the MMAs' 72 KB and the
# TMA's 48 KB, and the kernel is shared-memory-bandwidth bound (ncu: LSU
# wavefronts 76 % of peak, tensor pipe 51 % active).
FUSED_PRODUCER = False
# On CTA pairs (big leaf batches) form only S_r inside the kernel (paco_mm_tf32x3_fused_a):
# the A side's split launches go away, B^T stays pre-split.  Off: measured a wash on
# cfg5 (32.1-33.1 vs 32.0-32.9 ms; the leaf launches slow by ~8 %, the same as the
# 1.9 ms of A-side splits they save -- DESIGN.md section 5)
FUSED_A = False
# Leaf products on CTA pairs in the tf32 + 2 x bf16 format (paco_mm_tf32b2_multi):
# hi*hi on tf32, the hi*lo + lo*hi corrections as bf16 MMAs (a third less tensor
# time), bf16(hi) formed inside the kernel (TF32B2_CONVERT) so each operand element
# costs 6 bytes of L2 traffic instead of 8 -- the pair kernel is L2-bandwidth bound
# without it.  cfg5: 28.8 vs 32.9 ms (3xTF32), error vs f64 2.0e-5 vs 3.0e-5
# (DESIGN.md section 5).  False: 3xTF32 leaves.
TF32B2 = True
TF32B2_CONVERT = True
# ... and on plain fp32 operands (no split pass at all: S_r / T_r^T as quadrant views or
# one lincomb_multi pass per node side, B transposed once; the kernel forms both bf16
# parts): cfg5 23.8-25.4 ms vs 27.5-28.2 with the split pass (tools/cfg5_variants.py)
TF32B2_RAW = True
# ... or (the default where leaf blocks are a multiple of 8) in the bf16x3 format:
# S_r / T_r^T written as bf16 hi / lo planes by one paco_lincomb_split pass per node
# side, products hi*hi + hi*lo + lo*hi all on kind::f16 (paco_mm_bf16x3_multi): per CTA
# a 32-deep stage is 32 KB of TMA writes + 48 KB of MMA reads against 768 MMA clocks,
# so the leaves are tensor-bound instead of shared-memory bound
LEAF_BF16X3 = True
# ... with each leaf-level node's operands formed straight from the level-0 blocks (8-input
# paco_lincomb_split: S_r's quadrant q = the sum of its terms' quadrants q), so the level-1
# fp32 sums are never written or re-read
B3_DIRECT = True
# ... and B in its own k x m layout: T_r planes formed from B's quadrants, read by the MMA
# as MN-major tiles (paco_mm_bf16x3_multi_bn), so B is never transposed
B3_NATURAL = True
# ... with all 49 leaf operands of each side formed in ONE pass over A / B
# (paco_strassen_split49: every element read once, instead of once per term of its
# level-1 formula)
B3_ONEPASS = True


def _pair_batch(n: int, m: int, count: int) -> bool:
    """The library runs this 3xTF32 batch on CTA pairs (tc_gemm.cu tf32_pair)."""
    return ((n + 255) // 256) * ((m + 255) // 256) * count >= 3 * 74


def _strassen_dev(A: View, B: View, C: View, base: int, dtype: torch.dtype, stream) -> None:
    """C = A x B (square, power-of-two size) on one device, depth-first."""
    kid, dt = _RING[dtype]
    if C.rows <= base or C.rows % 2:
        launch_mm(kid, stream, A, B, C, overwrite=True)
        return
    h = C.rows // 2
    if kid == nat.SR_F32_TC and FUSED_COMBINE and (C.ld * 4) % 16 == 0 and C.ptr % 16 == 0:
        launch_fill(nat.SR_F32, stream, C)
        aligned = A.ptr % 16 == 0 and (A.ld * 4) % 16 == 0
        if aligned and B.ptr % 16 == 0 and (B.ld * 4) % 16 == 0 and _b3n_ok(C.rows, base, [(C, 1)]):
            _strassen_b3n(A, B, [(C, 1)], base, stream)
        elif TF32B2 and TF32B2_RAW and aligned and _b2raw_ok(C.rows, base):
            _strassen_tc_fused_t(A, _transpose(B, stream), [(C, 1)], base, stream, leaf=_default_leaf(C.rows, base))
        elif FUSED_PRODUCER and _fused_producer_ok(C.rows, base) and aligned:
            _strassen_tc_fused_t(A, _transpose(B, stream), [(C, 1)], base, stream)
        else:
            _strassen_tc_fused(A, B, [(C, 1)], base, stream)
        return
    if kid == nat.SR_F32_TC and (h <= base or h % 2) and h % 4 == 0:
        _leaf_level_tf32(A, B, C, stream)
        return
    ws = _Workspace(C.rows, dtype, C.device, A, B)
    _form(ws, A, B, dt, stream)
    for r in range(7):
        _strassen_dev(ws.S[r], ws.T[r], ws.M[r], base, dtype, stream)
    _combine(ws, C, dt, stream)


_STAGE_ALL = False  # test hook (set by tests/stage_all_check.py; see mm._REMOTE_ALL)


def _dtype_of_view(v: View) -> torch.dtype:
    return {4: torch.float32, 8: torch.float64}[v.elsize] if v.tensor is None or v.tensor.is_floating_point() \
        else v.tensor.dtype


def _local(v: View, dev: int, st) -> torch.Tensor:
    """A copy of (peer) view ``v`` in ``dev``'s memory, made on stream ``st``."""
    t = _local_empty(v, dev, st)
    es = t.element_size()
    nat.check(nat.load().paco_copy2d(dev, st.cuda_stream, t.data_ptr(), t.stride(0) * es, v.ptr, v.ld * es,
                                     v.cols * es, v.rows))
    return t


def _local_empty(v: View, dev: int, st) -> torch.Tensor:
    with torch.cuda.device(dev):
        t = torch.empty((v.rows, v.cols), dtype=_dtype_of_view(v), device=dev)
    t.record_stream(st)
    return t


def _copy_back(dst: View, t: torch.Tensor, dev: int, st) -> None:
    es = t.element_size()
    nat.check(nat.load().paco_copy2d(dev, st.cuda_stream, dst.ptr, dst.ld * es, t.data_ptr(), t.stride(0) * es,
                                     dst.cols * es, dst.rows))


def _ring_dtype(A, B) -> torch.dtype:
    dts = set()
    for x in (A, B):
        dts.add(x.dtype if isinstance(x, torch.Tensor) else {
            np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
            np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int64}[np.dtype(x.dtype)])
    if dts == {torch.float32}:
        return torch.float32
    if torch.float64 in dts or torch.float32 in dts:
        return torch.float64
    return torch.int64


def _staged_square(X, size: int, dtype: torch.dtype, dev: int) -> torch.Tensor:
    t = stage_in(X, dtype, dev)
    if t.shape[0] == size and t.shape[1] == size:
        return t
    out = torch.zeros((size, size), dtype=dtype, device=dev)
    out[:t.shape[0], :t.shape[1]] = t
    return out


def strassen_seq(A, B, n: int | None = None, base: int = DEFAULT_STRASSEN_BASE, *,
                 stream: torch.cuda.Stream | None = None):
    """C = A x B by Strassen down to ``base``, then classic MM.

    A, B: n x n NumPy arrays or CUDA tensors (float32 / float64 / int64 ring).
    Returns C of A's kind.
    """
    n = n if n is not None else A.shape[0]
    if tuple(A.shape) != (n, n) or tuple(B.shape) != (n, n):
        raise ValueError(f"shape mismatch: A{tuple(A.shape)} B{tuple(B.shape)} n={n}")
    dtype = _ring_dtype(A, B)
    dev = pick_device(A, B)
    size = _padded(n)
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(st):
            a = _staged_square(A, size, dtype, dev)
            b = _staged_square(B, size, dtype, dev)
            c = torch.empty((size, size), dtype=dtype, device=dev)
            _strassen_dev(View.of(a), View.of(b), View.of(c), base, dtype, st)
            c = c[:n, :n]
    if isinstance(A, np.ndarray):
        return c.cpu().numpy()
    return c if isinstance(A, torch.Tensor) and A.is_cuda else c.cpu()


def strassen_execute(plan: Plan, A, B, mode: str = "serial_sim", *, devices: list[int] | None = None,
                     with_report: bool = False):
    """Run a Strassen plan; returns C = A x B (and the
    CostReport -- work, makespan, temp_space_peak -- when ``with_report``).

    Workers map to ``devices[w % len(devices)]`` with one stream each.  S/T/M
    buffers live on the first device; FORM/COMBINE tasks run on their first
    worker, COMPUTE tasks run ``strassen_seq`` of their node into the
    parent's M slot; pieces of split leaves (``split_leftover``) write their
    cuboid of M (or of a k-cut temporary, folded by the leaf's REDUCE tasks).
    """
    meta = plan.meta
    if meta.get("algo") != "strassen":
        raise PlanError("not a Strassen plan")
    n, size, base = meta["n"], meta["n_padded"], meta["base"]
    if tuple(A.shape) != (n, n) or tuple(B.shape) != (n, n):
        raise ValueError(f"shape mismatch: A{tuple(A.shape)} B{tuple(B.shape)} n={n}")
    dtype = _ring_dtype(A, B)
    kid, dt = _RING[dtype]
    if devices is None:
        devices = [pick_device(A, B)]
    home = devices[0]
    dev_of = [devices[w % len(devices)] for w in range(plan.p)]
    for d in sorted(set(dev_of)):
        if d != home:
            nat.check(nat.load().paco_enable_peer(d, home))
    root: StrassenNode = meta["tree"]
    with torch.cuda.device(home):
        stage = torch.cuda.current_stream(home)
        a = _staged_square(A, size, dtype, home)
        b = _staged_square(B, size, dtype, home)
        c = torch.empty((size, size), dtype=dtype, device=home)
        # operand / output views of every node, and workspaces of internal nodes
        ops: dict[int, tuple[View, View, View]] = {id(root): (View.of(a), View.of(b), View.of(c))}
        wss: dict[int, _Workspace] = {}
        stack = [root]
        while stack:
            nd = stack.pop()
            if nd.kids:
                ws = _Workspace(nd.size, dtype, home, *ops[id(nd)][:2])
                wss[id(nd)] = ws
                for r, kid_nd in enumerate(nd.kids):
                    ops[id(kid_nd)] = (ws.S[r], ws.T[r], ws.M[r])
                    stack.append(kid_nd)
        # k-cut temporaries of leaves split across the workers (split_leftover)
        from .cuboid import temp_shape
        leaf_temps: dict[tuple[int, int], View] = {}
        by_leaf = {name: mp for name, mp in meta.get("split_leaves", {}).items()}
        for t in plan.tasks:
            if isinstance(t.region, LeafPiece) and t.region.cuboid.out and \
                    (id(t.region.node), t.region.cuboid.out) not in leaf_temps:
                bid = t.region.cuboid.out
                shp = temp_shape(by_leaf[str(t.region.node)], bid)
                leaf_temps[(id(t.region.node), bid)] = View.of(torch.empty(shp, dtype=dtype, device=home))
        staged = torch.cuda.Event()
        staged.record(stage)
        streams = [torch.cuda.Stream(device=dev_of[w]) for w in range(plan.p)]
        for s in streams:
            s.wait_event(staged)
        events: list = [None] * len(plan.tasks)
        by_name = {}
        stack = [root]
        while stack:
            nd = stack.pop()
            by_name[str(nd)] = nd
            stack.extend(nd.kids)

        def runner(task: Task) -> None:
            w = task.workers()[0]
            st = streams[w]
            for d in task.deps:
                st.wait_event(events[d])
            with torch.cuda.device(dev_of[w]):
                dv = dev_of[w]
                remote = dv != home or _STAGE_ALL
                if isinstance(task.region, LeafPiece):  # one worker's cuboid of a split leaf
                    leaf, cb = task.region.node, task.region.cuboid
                    A_n, B_n, C_n = ops[id(leaf)]
                    dst = C_n if cb.out == 0 else leaf_temps[(id(leaf), cb.out)]
                    a_v, b_v = A_n.sub(cb.i0, cb.l0, cb.n, cb.k), B_n.sub(cb.l0, cb.j0, cb.k, cb.m)
                    d_v = dst.sub(cb.out_i0, cb.out_j0, cb.n, cb.m)
                    if remote:  # operands over NVLink into local memory, the block back in one copy
                        a_l, b_l, c_l = _local(a_v, dv, st), _local(b_v, dv, st), _local_empty(d_v, dv, st)
                        launch_mm(kid, st, View.of(a_l), View.of(b_l), View.of(c_l), overwrite=True, device=dv)
                        _copy_back(d_v, c_l, dv, st)
                    else:
                        launch_mm(kid, st, a_v, b_v, d_v, overwrite=True, device=dv)
                elif isinstance(task.region, LeafFold):
                    f = task.region
                    A_n, B_n, C_n = ops[id(f.node)]
                    dst = C_n if f.out == 0 else leaf_temps[(id(f.node), f.out)]
                    src = leaf_temps[(id(f.node), f.temp)]
                    launch_fold(kid, st, dst.sub(f.oi, f.oj, f.n, f.m), src.sub(0, 0, f.n, f.m), False)
                elif task.kind == COMPUTE:
                    nd = task.region
                    A_n, B_n, C_n = ops[id(nd)]
                    with torch.cuda.stream(st):
                        if remote:  # the node's operands to this GPU, its product back in one copy
                            a_l, b_l, c_l = _local(A_n, dv, st), _local(B_n, dv, st), _local_empty(C_n, dv, st)
                            _strassen_dev(View.of(a_l), View.of(b_l), View.of(c_l), base, dtype, st)
                            _copy_back(C_n, c_l, dv, st)
                        else:
                            _strassen_dev(A_n, B_n, C_n, base, dtype, st)
                else:
                    what, name = task.region.split("[", 1)
                    nd = by_name[name[:-1]]
                    A_n, B_n, C_n = ops[id(nd)]
                    if what == "form":
                        _form(wss[id(nd)], A_n, B_n, dt, st)
                    else:
                        _combine(wss[id(nd)], C_n, dt, st)
            ev = torch.cuda.Event()
            ev.record(st)
            events[task.id] = ev

        report = execute_plan(plan, runner, mode)
        for s in streams:
            stage.wait_stream(s)
        out = c[:n, :n]
        torch.cuda.current_stream(home).synchronize()
    if isinstance(A, np.ndarray):
        out = out.cpu().numpy()
    elif not (isinstance(A, torch.Tensor) and A.is_cuda):
        out = out.cpu()
    return (out, report) if with_report else out

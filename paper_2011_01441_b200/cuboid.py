"""Iteration-space cuboids and the three PACO-MM partitioners.

The n x m x k iteration space of ``C (+)= A (x) B`` is cut into cuboids.  An
n or m cut splits the C face; a k cut gives both halves the same C face, so
the upper half writes a fresh temporary buffer and a REDUCE task folds it back
once both sides finished.  Reference behaviour followed (file:line in
/root/reference/pkg/src/paco/matmul.py):

* ``Cuboid``                  -- 60-91
* ``longest_axis``            -- 94-100 (ties n -> m -> k)
* cut tree / temps / reduces  -- 103-211 (``_CutNode``, ``_TempAlloc``,
  ``_split_cuboid``, ``_attach_reduces``, ``_finish_plan``)
* ``mm_paco_partition``       -- 214-243
* ``mm_one_piece_partition``  -- 246-300
* ``mm_hetero_partition``     -- 303-339

The same geometry is reused one level down (``csrc/cta_plan.cuh``, the
PACO CTA plan ``paco_plan_cta`` / ``PACO_MM_PACO_PLAN``) to spread one
device's cuboid over its 148 SMs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .plan import COMPUTE, REDUCE, Plan, PlanError, ProcList, Task, pruned_bfs_assign

DEFAULT_BASE = 32
AXES = ("n", "m", "k")


@dataclass(frozen=True)
class Cuboid:
    """Box [i0, i0+n) x [j0, j0+m) x [l0, l0+k); its C face lands in buffer
    ``out`` (0 = the caller's C, >0 = a temp) at (out_i0, out_j0)."""

    i0: int
    j0: int
    l0: int
    n: int
    m: int
    k: int
    out: int = 0
    out_i0: int = 0
    out_j0: int = 0

    @property
    def volume(self) -> int:
        return self.n * self.m * self.k

    @property
    def surface(self) -> int:
        return self.n * self.m + self.n * self.k + self.m * self.k

    def extent(self, axis: str) -> int:
        return {"n": self.n, "m": self.m, "k": self.k}[axis]

    def __str__(self) -> str:
        return "cuboid[i0=%d,j0=%d,l0=%d,n=%d,m=%d,k=%d,out=%d]" % (
            self.i0, self.j0, self.l0, self.n, self.m, self.k, self.out)


def longest_axis(n, m, k) -> str:
    """Name of the longest extent; ties prefer n, then m, then k."""
    if n >= m and n >= k:
        return "n"
    return "m" if m >= k else "k"


class _Node:
    """Node of the cut tree; leaves become COMPUTE tasks, k-cut nodes REDUCEs."""

    __slots__ = ("box", "axis", "kids", "temp", "task_id", "fold")

    def __init__(self, box: Cuboid):
        self.box = box
        self.axis: str | None = None
        self.kids: list[_Node] = []
        self.temp = 0
        self.task_id: int | None = None
        self.fold: tuple | None = None


class _Temps:
    """Numbers temporaries 1, 2, ... in allocation order; records n*m sizes."""

    def __init__(self):
        self.sizes: dict[int, int] = {}

    def new(self, n: int, m: int) -> int:
        tid = len(self.sizes) + 1
        self.sizes[tid] = n * m
        return tid

    @property
    def total(self) -> int:
        return sum(self.sizes.values())


def _cut(node: _Node, axis: str, left: int, temps: _Temps) -> list[_Node]:
    b = node.box
    length = b.extent(axis)
    if not 0 < left < length:
        raise PlanError(f"cut would create an empty extent on {axis}={length}")
    node.axis = axis
    if axis == "n":
        lo = Cuboid(b.i0, b.j0, b.l0, left, b.m, b.k, b.out, b.out_i0, b.out_j0)
        hi = Cuboid(b.i0 + left, b.j0, b.l0, b.n - left, b.m, b.k, b.out, b.out_i0 + left, b.out_j0)
    elif axis == "m":
        lo = Cuboid(b.i0, b.j0, b.l0, b.n, left, b.k, b.out, b.out_i0, b.out_j0)
        hi = Cuboid(b.i0, b.j0 + left, b.l0, b.n, b.m - left, b.k, b.out, b.out_i0, b.out_j0 + left)
    else:
        # the lower k half keeps the parent's C face, the upper half gets a temp
        node.temp = temps.new(b.n, b.m)
        lo = Cuboid(b.i0, b.j0, b.l0, b.n, b.m, left, b.out, b.out_i0, b.out_j0)
        hi = Cuboid(b.i0, b.j0, b.l0 + left, b.n, b.m, b.k - left, node.temp, 0, 0)
    node.kids = [_Node(lo), _Node(hi)]
    return node.kids


def _add_reduces(tasks: list[Task], root: _Node) -> None:
    """Postorder walk; every k-cut node appends one REDUCE after both sides."""

    def exits(node: _Node) -> tuple[int, ...]:
        if not node.kids:
            if node.task_id is None:
                raise PlanError("unassigned leaf in cut tree")
            return (node.task_id,)
        lo_ex = exits(node.kids[0])
        hi_ex = exits(node.kids[1])
        if node.axis != "k":
            return lo_ex + hi_ex
        both = lo_ex + hi_ex
        owners = sorted({w for tid in both for w in tasks[tid].workers()})
        b = node.box
        red = Task(
            id=len(tasks),
            kind=REDUCE,
            region=f"reduce[temp={node.temp}->out={b.out},n={b.n},m={b.m}]",
            worker=owners[0] if len(owners) == 1 else tuple(owners),
            deps=tuple(sorted(both)),
            cost_work=b.n * b.m,
        )
        tasks.append(red)
        node.task_id = red.id
        node.fold = (node.temp, b.out, b.out_i0, b.out_j0, b.n, b.m)
        return (red.id,)

    exits(root)


def _seal(tasks: list[Task], root: _Node, p: int, shape, temps: _Temps, variant: str,
          base: int) -> Plan:
    _add_reduces(tasks, root)
    folds = []
    stack = [root]
    while stack:  # preorder; order is irrelevant once sorted by task id
        node = stack.pop()
        if node.kids:
            if node.axis == "k":
                folds.append((node.task_id, list(node.fold)))
            stack.extend(reversed(node.kids))
    n, m, k = shape
    meta = {
        "algo": "mm",
        "variant": variant,
        "n": n,
        "m": m,
        "k": k,
        "base": base,
        "temp_sizes": dict(sorted(temps.sizes.items())),
        "temp_peak": temps.total,
        "reduces": dict(sorted(folds)),
    }
    return Plan(tasks=tasks, p=p, meta=meta)


def _check_extents(n: int, m: int, k: int) -> None:
    if min(n, m, k) < 1:
        raise PlanError("extents must be >= 1")


def mm_paco_partition(n: int, m: int, k: int, p: int, base: int = DEFAULT_BASE) -> Plan:
    """Multi-piece PACO-MM: pruned BFS over even halvings of the longest axis.

    Each worker receives a geometrically decreasing sequence of cuboids
    (matmul.py:214-243); leaves stop at max extent <= ``base``.
    """
    _check_extents(n, m, k)
    temps = _Temps()
    root = _Node(Cuboid(0, 0, 0, n, m, k))

    def halve(node: _Node) -> list[_Node]:
        b = node.box
        axis = longest_axis(b.n, b.m, b.k)
        return _cut(node, axis, b.extent(axis) // 2, temps)

    def small(node: _Node) -> bool:
        return max(node.box.n, node.box.m, node.box.k) <= base

    bfs = pruned_bfs_assign(root, 2, halve, small, p, cost=lambda nd: nd.box.volume)
    for t in bfs.tasks:
        t.region.task_id = t.id
    plan = _seal(bfs.tasks, root, p, (n, m, k), temps, "paco", base)
    for t in plan.tasks:
        if isinstance(t.region, _Node):
            t.region = t.region.box
    return plan


def _ratio_split(length: int, a: int, b: int) -> int:
    return max(1, length * a // (a + b))


def _quantized_split(length: int, a: int, b: int, q: int) -> int:
    """Cut ``length`` a:b on a multiple of ``q`` (keyword extension).

    A worker's kernel pays for whole tiles, so its cost is ceil(len / q); of the
    two multiples of q around the exact ratio point the one with the smaller
    max(cost_lo / a, cost_hi / b) wins (ties: the exact-ratio rounding).  Falls
    back to the reference split when the axis is shorter than two quanta.
    """
    exact = _ratio_split(length, a, b)
    if q <= 1 or length < 2 * q:
        return exact
    best = None
    for left in (max(q, exact // q * q), min(length - 1, -(-exact // q) * q)):
        if left <= 0 or left >= length:
            continue
        cost = max(-(-left // q) / a, -(-(length - left) // q) / b)
        key = (cost, abs(left - length * a / (a + b)))
        if best is None or key < best[0]:
            best = (key, left)
    return exact if best is None else best[1]


def mm_one_piece_partition(n: int, m: int, k: int, p: int, *, quantum: tuple[int, int, int] | None = None) -> Plan:
    """MM-1-Piece: exactly one cuboid per worker (matmul.py:250-300).

    The cut axis is whatever an evenly-halved *virtual* cuboid would cut; the
    real length is split floor(p/2):ceil(p/2), so prime p stays balanced.

    ``quantum=(qn, qm, qk)`` (keyword extension, not in the reference): cuts
    land on multiples of the kernel's tile / k quantum (``_quantized_split``),
    so no GPU-level cuboid ends in a partial C tile row or column -- the GPU
    level of the two-level plan then balances whole tiles, not elements.
    """
    _check_extents(n, m, k)
    quanta = dict(zip(AXES, quantum)) if quantum else None
    temps = _Temps()
    root = _Node(Cuboid(0, 0, 0, n, m, k))
    tasks: list[Task] = []

    def leaf(node: _Node, worker: int) -> None:
        node.task_id = len(tasks)
        tasks.append(Task(id=len(tasks), kind=COMPUTE, region=node.box, worker=worker,
                          cost_work=node.box.volume, label=1))

    def walk(node: _Node, procs: ProcList, virt: tuple) -> None:
        if len(procs) == 1:
            leaf(node, procs.first)
            return
        left_procs, right_procs = procs.split()
        axis = longest_axis(*virt)
        length = node.box.extent(axis)
        if length < 2:
            raise PlanError(
                f"extents too small to give every worker a nonempty piece (axis {axis})")
        a, b = len(left_procs), len(right_procs)
        left = _quantized_split(length, a, b, quanta[axis]) if quanta else _ratio_split(length, a, b)
        lo, hi = _cut(node, axis, left, temps)
        half = tuple(v / 2 if a == axis else v for a, v in zip(AXES, virt))
        walk(lo, left_procs, half)
        walk(hi, right_procs, half)

    walk(root, ProcList.range(p), (float(n), float(m), float(k)))
    return _seal(tasks, root, p, (n, m, k), temps, "one-piece", 0)


def mm_hetero_partition(n: int, m: int, k: int, weights: tuple[float, ...]) -> Plan:
    """One cuboid per worker, the longest real axis cut by summed throughput
    weights of the two worker halves (matmul.py:303-339)."""
    if not weights:
        raise PlanError("need at least one throughput weight")
    if any(w <= 0 for w in weights):
        raise PlanError("throughput weights must be positive")
    _check_extents(n, m, k)
    temps = _Temps()
    root = _Node(Cuboid(0, 0, 0, n, m, k))
    tasks: list[Task] = []

    def walk(node: _Node, procs: ProcList, wts: tuple) -> None:
        if len(procs) == 1:
            node.task_id = len(tasks)
            tasks.append(Task(id=len(tasks), kind=COMPUTE, region=node.box, worker=procs.first,
                              cost_work=node.box.volume, label=1))
            return
        left_procs, right_procs = procs.split()
        w_lo, w_hi = wts[:len(left_procs)], wts[len(left_procs):]
        b = node.box
        axis = longest_axis(b.n, b.m, b.k)
        length = b.extent(axis)
        s_lo, s_hi = sum(w_lo), sum(w_hi)
        left = min(max(int(length * s_lo / (s_lo + s_hi)), 1), length - 1)
        if length < 2:
            raise PlanError("weights too skewed for the available integer extents")
        lo, hi = _cut(node, axis, left, temps)
        walk(lo, left_procs, w_lo)
        walk(hi, right_procs, w_hi)

    walk(root, ProcList.range(len(weights)), tuple(float(w) for w in weights))
    return _seal(tasks, root, len(weights), (n, m, k), temps, "hetero", 0)


def temp_shape(plan: Plan, bid: int) -> tuple[int, int]:
    """(n, m) of temporary ``bid`` (matmul.py:465-469)."""
    for spec in plan.meta["reduces"].values():
        if spec[0] == bid:
            return (spec[4], spec[5])
    raise PlanError(f"temp buffer {bid} has no reduce")

"""CPU tests of the host-side PACO planner and engine.

Golden plans were produced by the reference itself (tests/golden/make_golden.py);
the examples below are the SPEC's known answers that
the survey verified against the reference code.
"""

import numpy as np
import pytest

from paper_2011_01441_b200 import (COMPUTE, REDUCE, Plan, PlanError, ProcList, Task, execute_plan,
                                   pruned_bfs_assign)
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200.plan import simulate_clocks


def _meta_json(meta):
    out = dict(meta)
    out["temp_sizes"] = {str(k): v for k, v in meta["temp_sizes"].items()}
    out["reduces"] = {str(k): list(v) for k, v in meta["reduces"].items()}
    return out


def test_golden_plans_byte_identical(golden_plans):
    fns = {"one_piece": M.mm_one_piece_partition, "paco": M.mm_paco_partition,
           "hetero": lambda n, m, k, w: M.mm_hetero_partition(n, m, k, tuple(w))}
    checked = 0
    for rec in golden_plans:
        fn = fns[rec["kind"]]
        if "error" in rec:
            with pytest.raises(PlanError) as ei:
                fn(*rec["args"])
            assert str(ei.value) == rec["error"]
            continue
        plan = fn(*rec["args"])
        assert plan.dump_text() == rec["dump"], rec["args"]
        assert _meta_json(plan.meta) == rec["meta"], rec["args"]
        checked += 1
    assert checked > 1500


def test_cfg1_plan_shape():
    plan = M.mm_paco_partition(384, 320, 256, 3)
    comp = plan.compute_tasks()
    assert len(comp) == 17 and sum(t.kind == REDUCE for t in plan.tasks) == 4
    vols = {w: sum(t.cost_work for t in comp if t.worker == w) for w in range(3)}
    assert vols == {0: 10490880, 1: 10490880, 2: 10475520}
    assert plan.meta["temp_sizes"] == {1: 30720, 2: 7680, 3: 7680, 4: 1920}


# --- SPEC examples (core) ----------------------------------------------------

def _binary_tree(depth):
    return ("node", depth)


def test_pruned_bfs_binary_p3():
    """Full binary tree of depth 3, p=3: 3 nodes at label 1, then 2 base nodes at label 2."""
    expand = lambda nd: [("node", nd[1] - 1)] * 2
    is_base = lambda nd: nd[1] == 0
    plan = pruned_bfs_assign(("node", 3), 2, expand, is_base, 3)
    labels = [t.label for t in plan.tasks]
    assert labels == [1, 1, 1, 2, 2]
    assert [t.worker for t in plan.tasks] == [0, 1, 2, 0, 1]


def test_pruned_bfs_arity7_p3():
    expand = lambda nd: [("node", nd[1] - 1)] * 7
    plan = pruned_bfs_assign(("node", 1), 7, expand, lambda nd: nd[1] == 0, 3)
    assert [t.label for t in plan.tasks] == [1, 1, 1, 2, 2, 2, 3]


def test_pruned_bfs_errors():
    with pytest.raises(PlanError):
        pruned_bfs_assign(0, 1, lambda x: [x, x], lambda x: True, 2)
    with pytest.raises(PlanError):
        pruned_bfs_assign(0, 2, lambda x: [x, x], lambda x: True, 0)
    with pytest.raises(PlanError, match="depth guard"):
        pruned_bfs_assign(0, 2, lambda x: [x, x], lambda x: False, 3, max_depth=5)
    with pytest.raises(PlanError, match="expected 2"):
        pruned_bfs_assign(0, 2, lambda x: [x], lambda x: False, 3)
    plan = pruned_bfs_assign("root", 2, lambda x: [x, x], lambda x: False, 1)
    assert len(plan.tasks) == 1 and plan.tasks[0].worker == 0


def test_execute_plan_cost_examples():
    chain = Plan([Task(0, COMPUTE, None, 0, (), 5), Task(1, COMPUTE, None, 0, (0,), 5),
                  Task(2, COMPUTE, None, 0, (1,), 5)], p=1)
    rep = execute_plan(chain)
    assert (rep.work_total, rep.work_max) == (15, 15)
    indep = Plan([Task(i, COMPUTE, None, i, (), 5) for i in range(4)], p=4)
    assert simulate_clocks(indep) == (20, 5)
    diamond = Plan([Task(0, COMPUTE, None, 0, (), 1), Task(1, COMPUTE, None, 0, (0,), 1),
                    Task(2, COMPUTE, None, 1, (0,), 1), Task(3, COMPUTE, None, 1, (1, 2), 1)], p=2)
    assert execute_plan(diamond).work_max == 3


def test_execute_plan_parallel_order_and_errors():
    plan = M.mm_paco_partition(64, 48, 80, 5)
    seen = []
    done = set()

    def runner(t):
        assert all(d in done for d in t.deps)
        seen.append(t.id)
        done.add(t.id)

    rep = execute_plan(plan, runner, "parallel")
    assert sorted(seen) == list(range(len(plan.tasks)))
    assert rep.wall_s is not None

    def bad(t):
        if t.id == 2:
            raise KeyError("boom")

    with pytest.raises(KeyError):
        execute_plan(plan, bad, "parallel")
    with pytest.raises(PlanError):
        execute_plan(plan, runner, "warp")


def test_plan_validate_errors():
    with pytest.raises(PlanError):
        Plan([Task(1, COMPUTE, None, 0)], p=1).validate()
    with pytest.raises(PlanError):
        Plan([Task(0, "nope", None, 0)], p=1).validate()
    with pytest.raises(PlanError):
        Plan([Task(0, COMPUTE, None, (0, 1))], p=2).validate()
    with pytest.raises(PlanError):
        Plan([Task(0, COMPUTE, None, 3)], p=2).validate()
    with pytest.raises(PlanError):
        Plan([Task(0, COMPUTE, None, 0, (0,))], p=1).validate()
    with pytest.raises(PlanError):
        ProcList(())
    with pytest.raises(PlanError):
        ProcList((2, 1))
    with pytest.raises(PlanError):
        ProcList.range(1).split()
    assert ProcList.range(5).split() == (ProcList((0, 1)), ProcList((2, 3, 4)))


# --- SPEC examples (matmul partitioners) --------------------------------------

def test_one_piece_examples():
    p2 = M.mm_one_piece_partition(8, 4, 2, 2)
    assert [(t.region.n, t.region.m, t.region.k) for t in p2.tasks] == [(4, 4, 2), (4, 4, 2)]
    p3 = M.mm_one_piece_partition(9, 4, 2, 3)
    assert [t.cost_work for t in p3.compute_tasks()] == [24, 24, 24]
    p5 = M.mm_one_piece_partition(32, 32, 32, 5)
    assert len(p5.compute_tasks()) == 5
    with pytest.raises(PlanError):
        M.mm_one_piece_partition(2, 1, 1, 3)


def test_hetero_examples():
    plan = M.mm_hetero_partition(16, 4, 4, (3, 1))
    assert [t.region.n for t in plan.tasks] == [12, 4]
    assert M.mm_hetero_partition(8, 4, 2, (1, 1)).dump_text() == \
        M.mm_one_piece_partition(8, 4, 2, 2).dump_text()
    with pytest.raises(PlanError):
        M.mm_hetero_partition(8, 8, 8, ())
    with pytest.raises(PlanError):
        M.mm_hetero_partition(8, 8, 8, (1, 0))


def test_paco_examples():
    plan = M.mm_paco_partition(8, 8, 8, 3, base=1)
    lab1 = [t for t in plan.compute_tasks() if t.label == 1]
    assert len(lab1) == 3 and all(t.cost_work == 8 ** 3 // 4 for t in lab1)
    assert len(M.mm_paco_partition(8, 8, 8, 1).tasks) == 1


@pytest.mark.parametrize("p", [1, 2, 3, 5, 7, 12, 13])
def test_partitions_tile_the_cuboid(p):
    rng = np.random.default_rng(p)
    for _ in range(20):
        n, m, k = (int(x) for x in rng.integers(1, 70, 3))
        for fn in (M.mm_paco_partition, M.mm_one_piece_partition):
            try:
                plan = fn(n, m, k, p)
            except PlanError:
                continue
            cover = np.zeros((n, m, k), np.int32)
            for t in plan.compute_tasks():
                c = t.region
                cover[c.i0:c.i0 + c.n, c.j0:c.j0 + c.m, c.l0:c.l0 + c.k] += 1
            assert (cover == 1).all()


def test_one_piece_balance_primes():
    """Perfect-strong-scaling check (SPEC acceptance 4): work_max <= 1.10 work_total / p."""
    for p in (2, 3, 5, 7, 13):
        plan = M.mm_one_piece_partition(512, 512, 512, p)
        rep = execute_plan(plan)
        assert rep.work_max <= 1.10 * rep.work_total / p


# --- native CTA-level planner == reference rule -----------------------------

def test_native_one_piece_matches_reference_rule():
    rng = np.random.default_rng(3)
    shapes = [(8192, 8192, 8192), (16384, 16384, 16384), (65536, 1024, 256), (384, 320, 256)]
    shapes += [tuple(int(x) for x in rng.integers(1, 3000, 3)) for _ in range(40)]
    for (n, m, k) in shapes:
        for p in (1, 2, 3, 5, 7, 8, 13, 148, 296):
            try:
                plan = M.mm_one_piece_partition(n, m, k, p)
            except PlanError:
                with pytest.raises(PlanError):
                    nat.plan_one_piece(n, m, k, p)
                continue
            want = [(t.region.i0, t.region.j0, t.region.l0, t.region.n, t.region.m, t.region.k)
                    for t in plan.compute_tasks()]
            assert nat.plan_one_piece(n, m, k, p) == want, (n, m, k, p)


def test_cta_plan_balance_and_cover():
    """Default CTA-level plan: tiles the unit grid exactly and stays within 3% of V/p."""
    for (n, m, k) in [(8192, 8192, 8192), (16384, 16384, 16384), (9363, 8192, 8192),
                      (7021, 10923, 8192), (4096, 4096, 4096), (65536, 1024, 256)]:
        bm, bn, kq, cps = nat.tile_shape(nat.SR_MINPLUS_SAT32)
        p = 148 * cps
        pieces = nat.plan_cta(nat.SR_MINPLUS_SAT32, n, m, k, p)
        units = (-(-n // bm), -(-m // bn), -(-k // kq))
        vols = np.array([pc[3] * pc[4] * pc[5] for pc in pieces], dtype=float)
        assert vols.sum() == units[0] * units[1] * units[2]
        assert vols.max() / vols.mean() < 1.05, (n, m, k, vols.max() / vols.mean())
        if (n, m, k) == (8192, 8192, 8192):
            assert vols.max() / vols.mean() < 1.015
    small = nat.plan_cta(nat.SR_MINPLUS_SAT32, 300, 260, 515, 7)
    cover = np.zeros((3, 3, 129), np.int32)
    for a, b, c, dn, dm, dk in small:
        cover[a:a + dn, b:b + dm, c:c + dk] += 1
    assert (cover == 1).all()


def test_cta_grid_plan_tiles_iteration_space_once():
    """Default tile-grid plan: every (C tile, k quantum) cell covered exactly once."""
    for sr in (nat.SR_MINPLUS_SAT32, nat.SR_INT_I64):
        bm, bn, kq, _ = nat.tile_shape(sr)
        for (n, m, k) in [(300, 260, 515), (1000, 700, 9000), (129, 4000, 64), (1, 1, 1), (200, 150, 3000)]:
            s, ctas = nat.cta_grid(sr, n, m, k)
            units = (-(-n // bm), -(-m // bn), -(-k // kq))
            assert ctas == units[0] * units[1] * s and 1 <= s <= units[2]
            cover = np.zeros(units, np.int32)
            for a, b, c, dn, dm, dk in nat.grid_pieces(sr, n, m, k):
                assert dk >= 1
                cover[a:a + dn, b:b + dm, c:c + dk] += 1
            assert (cover == 1).all()


@pytest.mark.parametrize("p", [1, 2, 3, 5, 6, 7, 8, 13])
def test_quantized_one_piece_plan(p):
    """quantum= (keyword extension): cuts on tile multiples, the cuboid still tiled
    exactly once, and the max per-worker whole-tile cost never worse than the
    reference cut's (the GPU level of bench.py --gpus N)."""
    rng = np.random.default_rng(p)
    shapes = [(8192, 8192, 8192), (16384, 16384, 16384), (65536, 1024, 256), (3000, 5000, 700)]
    shapes += [tuple(int(x) for x in rng.integers(300, 9000, 3)) for _ in range(6)]
    q = (128, 128, 4)
    for (n, m, k) in shapes:
        ref = M.mm_one_piece_partition(n, m, k, p)
        pl = M.mm_one_piece_partition(n, m, k, p, quantum=q)
        pl.validate()
        regs = [t.region for t in pl.tasks if t.kind == COMPUTE]
        assert len(regs) == p
        vol = sum(r.n * r.m * r.k for r in regs)
        assert vol == n * m * k
        for r in regs:
            for ax, (o, full) in enumerate(((r.i0, n), (r.j0, m), (r.l0, k))):
                # every cut lands on a quantum unless the axis is shorter than two quanta
                assert o % q[ax] == 0 or full < 2 * q[ax], (n, m, k, p, r)

        def worst(plan):
            return max(-(-t.region.n // 128) * -(-t.region.m // 128) * t.region.k
                       for t in plan.tasks if t.kind == COMPUTE)
        assert worst(pl) <= worst(ref) * 1.02, (n, m, k, p, worst(pl), worst(ref))


@pytest.mark.parametrize("n", [512, 1000, 4096, 8192, 16384, 65536])
def test_host_pipeline_row_blocks(n):
    """mm_seq's last-phase row blocks (host logic): they tile [0, n) in order, on
    128-row boundaries except the end, shrink toward the end (geometric schedule)
    and end with a small block, so only a small download is exposed."""
    from paper_2011_01441_b200 import mm as MMmod
    e = MMmod._row_edges(n)
    assert e[0] == 0 and e[-1] == n and all(b > a for a, b in zip(e, e[1:]))
    assert all(x % 128 == 0 for x in e[:-1])
    sizes = [b - a for a, b in zip(e, e[1:])]
    if MMmod._ROW_DECAY is not None and n >= 4096:
        assert sizes[-1] == 128 + n % 128
        assert all(a >= b for a, b in zip(sizes[1:], sizes[2:]))
        assert max(sizes) <= 2 * MMmod._ROW_CAP

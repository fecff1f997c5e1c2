"""CPU tests of the PACO-Strassen planners."""

import math

import pytest

from paper_2011_01441_b200 import COMPUTE, MERGE, PlanError, execute_plan
from paper_2011_01441_b200.strassen import (SuperRoundCfg, strassen_const_pieces_partition,
                                            strassen_paco_partition)


def computes(plan):
    return [t for t in plan.tasks if t.kind == COMPUTE]


def test_p1_is_sequential():
    plan = strassen_paco_partition(1024, 1, base=64)
    assert len(plan.tasks) == 1 and plan.tasks[0].kind == COMPUTE and plan.tasks[0].worker == 0


def test_p7_one_node_per_worker():
    plan = strassen_paco_partition(1024, 7, base=64)
    c = computes(plan)
    assert sorted(t.worker for t in c) == list(range(7))
    assert all(t.region.depth == 1 and t.label == 1 for t in c)
    kinds = [t.kind for t in plan.tasks]
    assert kinds.count(MERGE) == 2  # root FORM + root COMBINE


def test_p3_batch_rule():
    plan = strassen_paco_partition(1024, 3, base=64)
    c = computes(plan)
    d1 = [t for t in c if t.region.depth == 1]
    assert [t.label for t in d1] == [1, 1, 1, 2, 2, 2]
    # the 7th depth-1 node expanded: 7 depth-2 nodes -> batches of 3, 3 and a straggler
    d2 = [t for t in c if t.region.depth >= 2]
    assert len(d2) >= 7


def test_plan_is_valid_dag_and_covers_tree():
    for p in (1, 2, 3, 5, 6, 7, 8, 13):
        for plan in (strassen_paco_partition(2 ** 12, p, base=256),
                     strassen_const_pieces_partition(2 ** 12, p, SuperRoundCfg(2), base=256)):
            plan.validate()
            c = computes(plan)
            # total computed volume == 7^log2(n / base) leaves of base-size work, exactly
            vol = sum(t.cost_work for t in c)
            assert vol == 7 ** 12
            rep = execute_plan(plan)
            assert rep.work_max >= rep.work_total / p


def test_const_pieces_gamma1_p3():
    plan = strassen_const_pieces_partition(1024, 3, SuperRoundCfg(1), base=64)
    c = computes(plan)
    assert len(c) == 7 and all(t.region.depth == 1 for t in c)
    per = {w: sum(1 for t in c if t.worker == w) for w in range(3)}
    assert max(per.values()) == 3


def test_const_pieces_large_gamma_equals_paco():
    a = strassen_paco_partition(2 ** 10, 3, base=8)
    b = strassen_const_pieces_partition(2 ** 10, 3, SuperRoundCfg(64), base=8)
    assert [str(t.region) for t in computes(a)] == [str(t.region) for t in computes(b)]


def test_const_pieces_balance_gamma8():
    """SPEC acceptance 2: p=3, gamma=8, n=2^12 -> (max-min)/max < 1%."""
    plan = strassen_const_pieces_partition(2 ** 12, 3, SuperRoundCfg(8), base=1)
    per = [0, 0, 0]
    for t in computes(plan):
        per[t.worker] += t.cost_work
    assert (max(per) - min(per)) / max(per) < 0.01


def test_temp_bound():
    """Temp space before first assignment <= 21 n^2 sum (7/4)^i (Theorem strassen proof)."""
    n = 2 ** 12
    for p in (2, 3, 7, 8):
        plan = strassen_paco_partition(n, p, base=64)
        bound = 21 * n * n * sum((7 / 4) ** i for i in range(math.ceil(math.log(p, 7)) + 1))
        # the plan's workspace holds S/T/M of every internal node; nodes below the
        # first assignment depth add a geometrically smaller term
        assert plan.meta["temp_peak"] <= 2 * bound


def test_errors():
    with pytest.raises(PlanError):
        SuperRoundCfg(0)
    with pytest.raises(PlanError):
        strassen_paco_partition(0, 2)
    with pytest.raises(PlanError):
        strassen_const_pieces_partition(64, 0)


@pytest.mark.parametrize("p", [5, 6, 8])
def test_split_leftover_balances_cfg5(p):
    """the leftover base leaves, cut into p MM-1-Piece cuboids,
    remove the 87.5 % (p = 8) / 90.7 % (p = 6) efficiency cap of cfg5's plan."""
    from paper_2011_01441_b200.strassen import LeafPiece, LeafFold, strassen_paco_partition as part
    loads = {}
    for split in (False, True):
        plan = part(16384, p, base=4096, split_leftover=split)
        plan.validate()
        w = [0] * p
        for t in plan.tasks:
            if t.kind in ("compute", "reduce"):
                w[t.workers()[0]] += t.cost_work
        loads[split] = max(w) / (sum(w) / p)
    assert loads[True] < 1.001 and loads[True] < loads[False]
    assert loads[False] > (1.05 if p != 5 else 1.01)
    plan = part(16384, p, base=4096, split_leftover=True)
    pieces = [t.region for t in plan.tasks if isinstance(t.region, LeafPiece)]
    leaves = {str(pc.node) for pc in pieces}
    for name in leaves:  # each split leaf's cuboids tile its 4096^3 cube exactly once
        vol = sum(pc.cuboid.n * pc.cuboid.m * pc.cuboid.k for pc in pieces if str(pc.node) == name)
        assert vol == 4096 ** 3
    folds = [t for t in plan.tasks if isinstance(t.region, LeafFold)]
    assert all(t.kind == "reduce" for t in folds)
    assert "split" in plan.meta["variant"]


def test_split_leftover_noop_when_even():
    from paper_2011_01441_b200.strassen import strassen_paco_partition as part
    a, b = part(16384, 7, base=4096), part(16384, 7, base=4096, split_leftover=True)
    assert a.dump_text() == b.dump_text()

"""Per-worker kernel time of GPU-level PACO plans, measured one worker at a time
on one B200 (cfg4 by default): t_p = max over workers of the time its cuboids
take alone (k-cut folds fused, as the multi-GPU executors run them), and the
compute-only strong-scaling efficiency E(p) = t_1 / (p * t_p) the plan allows
(SURVEY.md 8(d) cfg4).  Communication is not included (one GPU here)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm, fold_destinations

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,4,5,7,8").split(",")]
which = sys.argv[3] if len(sys.argv) > 3 else "maxplus"
g = torch.Generator(device="cuda").manual_seed(1004)
if which == "maxplus":
    sr, kid, lo, zero = M.SEMIRING_MAXPLUS, nat.SR_MAXPLUS_SAT32, -2**20, -2**30
else:
    sr, kid, lo, zero = M.SEMIRING_MINPLUS_SAT, nat.SR_MINPLUS_SAT32, 0, 2**30
A = torch.randint(lo, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
B = torch.randint(lo, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
C = torch.full((n, n), zero, device="cuda", dtype=torch.int32)
a, b, c = View.of(A), View.of(B), View.of(C)
st = torch.cuda.current_stream()


def timed(fn, reps=2):
    fn(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {"n": n, "semiring": which + "_sat32", "plans": []}
t1 = None
for p in ps:
    # QUANTUM=1: GPU-level cuts on tile multiples (the plan bench.py --gpus N runs)
    plan = M.mm_one_piece_partition(n, n, n, p, quantum=nat.tile_shape(kid)[:3] if os.environ.get("QUANTUM") == "1" else None)
    dest = fold_destinations(plan)
    per_worker = []
    for w in range(p):
        tasks = [t for t in plan.tasks if t.kind == "compute" and t.worker == w]

        def run():
            for t in tasks:
                cb = t.region
                _, fi, fj = dest.get(cb.out, (0, 0, 0))
                launch_mm(kid, st, a.sub(cb.i0, cb.l0, cb.n, cb.k), b.sub(cb.l0, cb.j0, cb.k, cb.m),
                          c.sub(fi + cb.out_i0, fj + cb.out_j0, cb.n, cb.m), flags=nat.MM_ATOMIC)
        per_worker.append(timed(run))
    tp = max(per_worker)
    t1 = tp if p == 1 else t1
    row = {"p": p, "t_p_ms": tp, "worker_ms": per_worker,
           "efficiency": (t1 / (p * tp)) if t1 else None,
           "reduces": sum(1 for t in plan.tasks if t.kind == "reduce")}
    out["plans"].append(row)
    print(f"p={p}: t_p {tp:8.2f} ms  E(p) {row['efficiency']:.3f}  workers {[round(x, 1) for x in per_worker]}",
          flush=True)
json.dump(out, open(os.environ.get("OUT", "gpurun_out/worker_times.json"), "w"), indent=1)

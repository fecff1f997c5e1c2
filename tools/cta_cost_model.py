"""Processor-sharing simulation of a CTA plan on 148 SMs x 2 slots; calibrates
the per-tile-visit overhead against measured kernel times (dev tool)."""
import sys, os, heapq
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_01441_b200 import _native as nat

def simulate(costs, sms=148, slots=2):
    # each SM runs its active CTAs at a shared total rate 1
    nxt = 0
    active = [[] for _ in range(sms)]
    for s in range(slots):
        for sm in range(sms):
            if nxt < len(costs):
                active[sm].append(costs[nxt]); nxt += 1
    t = 0.0
    while any(active):
        # time until first completion
        dt = min(min(a) * len(a) for a in active if a)
        t += dt
        for sm in range(sms):
            a = active[sm]
            if not a:
                continue
            d = dt / len(a)
            a[:] = [x - d for x in a]
            done = [x for x in a if x <= 1e-9]
            a[:] = [x for x in a if x > 1e-9]
            for _ in done:
                if nxt < len(costs):
                    a.append(costs[nxt]); nxt += 1
    return t

def est(n, m, k, p, ovh):
    bm, bn, kq, cps = nat.tile_shape(nat.SR_MINPLUS_SAT32)
    pcs = nat.plan_cta(nat.SR_MINPLUS_SAT32, n, m, k, p)
    costs = [q[3] * q[4] * (min(q[5] * kq, k - q[2] * kq) + ovh) for q in pcs]
    return simulate(costs)

if __name__ == "__main__":
    ovh = float(sys.argv[1])
    for spec in sys.argv[2:]:
        n, m, k = (int(x) for x in spec.split("x"))
        print(spec, " ".join(f"p={p}:{est(n, m, k, p, ovh):.0f}" for p in (1184, 2048, 4096, 8192)))

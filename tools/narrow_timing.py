"""Time the reference's int64 SEMIRING_MINPLUS / SEMIRING_INT at 8192^3 through mm_seq
(device-resident int64 operands, narrowed to the 32-bit kernels) vs the SAT kernel."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import matmul as M


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randint(0, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
b = torch.randint(0, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
c = torch.full((n, n), 2**30, device="cuda", dtype=torch.int32)
ops = 2 * n ** 3
res = {}
res["sat32_ms"] = timed(lambda: M.mm_seq(a, b, c, M.SEMIRING_MINPLUS_SAT))
a64, b64 = a.long(), b.long()
c64 = torch.full((n, n), 2**62, device="cuda", dtype=torch.int64)
res["minplus_i64_narrowed_ms"] = timed(lambda: M.mm_seq(a64, b64, c64, M.SEMIRING_MINPLUS))
res["int_i64_narrowed_ms"] = timed(lambda: M.mm_seq(a64 - 2**19, b64 - 2**19, c64, M.SEMIRING_INT))
# 10 % INF = 2^62 sentinels in both operands: still the u32 kernel (INF-keeping code)
ai, bi = a64.clone(), b64.clone()
ai[torch.rand(ai.shape, device="cuda", generator=g) < 0.1] = 2**62
bi[torch.rand(bi.shape, device="cuda", generator=g) < 0.1] = 2**62
res["minplus_i64_inf10_ms"] = timed(lambda: M.mm_seq(ai, bi, c64, M.SEMIRING_MINPLUS))
del ai, bi
a64[0, 0] = -1  # a negative operand: the int64 kernel
res["minplus_i64_wide_ms"] = timed(lambda: M.mm_seq(a64, b64, c64, M.SEMIRING_MINPLUS), reps=1)
for k in list(res):
    res[k.replace("_ms", "_top_s")] = ops / res[k] / 1e9
res["ratio_narrowed_vs_sat"] = res["sat32_ms"] / res["minplus_i64_narrowed_ms"]
print(json.dumps(res, indent=1))

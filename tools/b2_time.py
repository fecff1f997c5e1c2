"""Time one paco_mm_tf32b2_multi batch (7 x 4096^3) -- with PACO_LIB pointing at an
ablated build, the L2-bandwidth hypothesis of the pair kernel can be checked."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat

lib = nat.load()
n = m = k = 4096
cnt = 7
st = torch.cuda.current_stream().cuda_stream
ops = []
for _ in range(2 * cnt):
    ops.append((torch.rand(n, k, device="cuda"), torch.rand(n, k, device="cuda").to(torch.bfloat16),
                torch.rand(n, k, device="cuda").to(torch.bfloat16)))
C = torch.zeros(n, m, device="cuda")
arr = lambda xs: (ctypes.c_void_p * cnt)(*[x.data_ptr() for x in xs])  # noqa: E731
ndst = (ctypes.c_int32 * cnt)(*[1] * cnt)
dst = (ctypes.c_void_p * (4 * cnt))(*([C.data_ptr(), 0, 0, 0] * cnt))
sign = (ctypes.c_int32 * (4 * cnt))(*([1, 1, 1, 1] * cnt))
A, B = ops[:cnt], ops[cnt:]
fn = lambda: nat.check(lib.paco_mm_tf32b2_multi(0, st, cnt, arr([x[0] for x in A]), arr([x[1] for x in A]),  # noqa: E731
                                                arr([x[2] for x in A]), k, arr([x[0] for x in B]),
                                                arr([x[1] for x in B]), arr([x[2] for x in B]), k, ndst, dst, sign,
                                                m, n, m, k))
cv = os.environ.get("CV") == "1"
if cv:
    fn = lambda: nat.check(lib.paco_mm_tf32b2_multi(0, st, cnt, arr([x[0] for x in A]), None,  # noqa: E731
                                                    arr([x[2] for x in A]), k, arr([x[0] for x in B]), None,
                                                    arr([x[2] for x in B]), k, ndst, dst, sign, m, n, m, k))
fn()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"lib": os.environ.get("PACO_LIB", "default"), "cv": cv, "ms": sorted(ts)}))

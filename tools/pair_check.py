"""CTA-pair 3xTF32 path (tf32_pair) correctness and cfg5 timing.

    python tools/pair_check.py            # default selection (pairs for big batches)
    PACO_DEV_KNOBS=1 PACO_TF32_PAIR=0 python tools/pair_check.py   # single-CTA kernels
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import strassen as S

lib = nat.load()
res = {"pair_knob": os.environ.get("PACO_TF32_PAIR")}
g = torch.Generator(device="cuda").manual_seed(0)
st = torch.cuda.current_stream().cuda_stream
for (n, m, k, cnt, multi) in ((4096, 4096, 4096, 7, False), (4096, 4096, 4096, 7, True), (3000, 2600, 1040, 8, True)):
    a = [torch.rand(n, k, device="cuda", generator=g) * 2 - 1 for _ in range(cnt)]
    b = [torch.rand(m, k, device="cuda", generator=g) * 2 - 1 for _ in range(cnt)]   # B^T
    hi_lo = []
    for x in a + b:
        h, l = torch.empty_like(x), torch.empty_like(x)
        nat.check(lib.paco_tf32_split(0, st, 1, (ctypes.c_void_p * 1)(x.data_ptr()), (ctypes.c_int64 * 1)(x.shape[1]),
                                      (ctypes.c_int32 * 1)(1), x.shape[0], x.shape[1], 0, h.data_ptr(), l.data_ptr(),
                                      x.shape[1]))
        hi_lo.append((h, l))
    arr = lambda xs: (ctypes.c_void_p * cnt)(*[x.data_ptr() for x in xs])  # noqa: E731
    ah, al = arr([p[0] for p in hi_lo[:cnt]]), arr([p[1] for p in hi_lo[:cnt]])
    bh, bl = arr([p[0] for p in hi_lo[cnt:]]), arr([p[1] for p in hi_lo[cnt:]])
    C = [torch.zeros(n, m, device="cuda") for _ in range(2)]
    if multi:   # product q folds into C[q % 2] with sign +1 and C[(q + 1) % 2] with sign -1 (q odd)
        ndst = (ctypes.c_int32 * cnt)(*[2] * cnt)
        dst = (ctypes.c_void_p * (4 * cnt))()
        sign = (ctypes.c_int32 * (4 * cnt))()
        for q in range(cnt):
            dst[4 * q], dst[4 * q + 1] = C[q % 2].data_ptr(), C[(q + 1) % 2].data_ptr()
            sign[4 * q], sign[4 * q + 1] = 1, (-1 if q % 2 else 1)
        fn = lambda: nat.check(lib.paco_mm_tf32x3_multi(0, st, cnt, ah, al, k, bh, bl, k, ndst, dst, sign, m, n, m, k))  # noqa: E731
    else:
        outs = [torch.zeros(n, m, device="cuda") for _ in range(cnt)]
        fn = lambda: nat.check(lib.paco_mm_tf32x3(0, st, cnt, ah, al, k, bh, bl, k, arr(outs), m, n, m, k,  # noqa: E731
                                                  nat.MM_OVERWRITE))
    fn()
    torch.cuda.synchronize()
    if multi:
        ref = [torch.zeros(n, m, dtype=torch.float64, device="cuda") for _ in range(2)]
        for q in range(cnt):
            p = a[q].double() @ b[q].double().t()
            ref[q % 2] += p
            ref[(q + 1) % 2] += (-p if q % 2 else p)
        err = max(float((C[i].double() - ref[i]).norm() / ref[i].norm()) for i in range(2))
    else:
        err = max(float((outs[q].double() - a[q].double() @ b[q].double().t()).norm() /
                        (a[q].double() @ b[q].double().t()).norm()) for q in range(cnt))
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    flop = 3 * 2.0 * n * m * k * cnt
    res[f"{n}x{m}x{k}x{cnt}{'_multi' if multi else ''}"] = {"rel_err": err, "ms": min(ts),
                                                             "tf32_tflops": flop / min(ts) / 1e9}
    print(json.dumps(res), flush=True)
n = 16384
a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
for _ in range(2):
    c = S.strassen_seq(a, b, n, base=n // 4)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = S.strassen_seq(a, b, n, base=n // 4)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
with nat.kernel_timing() as kt:
    S.strassen_seq(a, b, n, base=n // 4)
    torch.cuda.synchronize()
    tc = kt.read(nat.KT_TC_GEMM)
rows = torch.arange(0, n, n // 64, device="cuda")
ref = a[rows].double() @ b.double()
res["cfg5"] = {"ms": sorted(ts), "tc_ms_launches": tc,
               "rel_err_rows": float((c[rows].double() - ref).norm() / ref.norm())}
print(json.dumps(res, indent=1))

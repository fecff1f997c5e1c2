"""Quick check + timing of the bf16 tcgen05 path for the library in PACO_LIB
(kernel-configuration experiments, tools/build_variant.sh).

cfg3 (65536x1024x256, overwrite and accumulate) against torch.mm, and the
streaming 8192^3 bf16 GEMM; prints one JSON line.
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    best = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        best.append(e0.elapsed_time(e1) / reps * 1e3)
    return sorted(best)[1]


def main():
    g = torch.Generator(device="cuda").manual_seed(3)
    st = torch.cuda.current_stream()
    out = {"lib": os.environ.get("PACO_LIB", "default")}
    for name, (n, k, m) in (("cfg3", (65536, 256, 1024)), ("sq8192", (8192, 8192, 8192))):
        a = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
        b = torch.randn(k, m, device="cuda", generator=g).to(torch.bfloat16)
        c = torch.empty(n, m, device="cuda")
        ref = torch.mm(a.float(), b.float())
        launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
        err = float((c - ref).abs().max() / ref.abs().max())
        c2 = torch.ones(n, m, device="cuda")
        launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c2))
        err2 = float((c2 - 1 - ref).abs().max() / ref.abs().max())
        us = timed(lambda: launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True),
                   20 if name == "cfg3" else 5)
        byts = 2 * n * k + 2 * k * m + 4 * n * m
        out[name] = {"us": us, "err": err, "err_acc": err2, "tb_s": byts / us / 1e6,
                     "tflop_s": 2 * n * m * k / us / 1e6}
        del a, b, c, c2, ref
    print(json.dumps(out))


if __name__ == "__main__":
    main()

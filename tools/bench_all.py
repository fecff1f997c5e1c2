"""Device-resident timing of all five BASELINE configs on one B200 (dev report).

bench.py is the driver contract (cfg2 headline); this tool reports every
config with its roofline so DESIGN.md / profiles/ can cite one run.  Inputs
follow SURVEY.md 8(d) (seeded, generated on the device with the same
distributions; correctness is covered by tests/).  Each number is the median
of K back-to-back launches between CUDA events after warm-up.

    python tools/bench_all.py [--reps 5] [--out profiles/bench_all.json]
"""

import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import strassen as S
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else {}
HBM = PEAKS.get("hbm_gbs", 6554.9)
SM_MAX_MHZ = PEAKS.get("sm_max_mhz", 1965.0)


def timed(fn, reps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out), min(out)


def probe(which):
    tpc, mhz = ctypes.c_double(), ctypes.c_double()
    nat.check(nat.load().paco_alu_probe(0, None, which, 20000, ctypes.byref(tpc), ctypes.byref(mhz)))
    return tpc.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="1,2,3,4,5")
    args = ap.parse_args()
    only = {int(x) for x in args.only.split(",")}
    g = torch.Generator(device="cuda").manual_seed(2011)
    st = torch.cuda.current_stream()
    res = {}
    tpc_min = probe(0)
    tpc_ffma = probe(2)
    alu_peak = 2 * tpc_min * 148 * SM_MAX_MHZ / 1e6      # Top/s at max clock
    ffma_peak = 2 * tpc_ffma * 148 * SM_MAX_MHZ / 1e6    # TFLOP/s at max clock
    res["probes"] = {"viaddmnmx_terms_per_clk_sm": tpc_min, "ffma_terms_per_clk_sm": tpc_ffma,
                     "alu_peak_top_s": alu_peak, "ffma_peak_tflop_s": ffma_peak,
                     "sm_max_mhz": SM_MAX_MHZ, "hbm_gbs": HBM}

    if 1 in only:  # cfg1: (+,x) int32 -> int64, 384x256x320, PACO p=3 (3 streams)
        a = torch.randint(-8, 9, (384, 256), device="cuda", dtype=torch.int32, generator=g)
        b = torch.randint(-8, 9, (256, 320), device="cuda", dtype=torch.int32, generator=g)
        c = torch.zeros(384, 320, device="cuda", dtype=torch.int64)
        plan = M.mm_paco_partition(384, 320, 256, 3)
        med, best = timed(lambda: M.mm_execute(plan, a, b, c, M.SEMIRING_INT), args.reps)
        one, _ = timed(lambda: launch_mm(nat.SR_INT_I32_I64, st, View.of(a), View.of(b), View.of(c)), args.reps)
        ops = 2 * 384 * 320 * 256
        res["cfg1"] = {"ms_paco_p3_mm_execute": med, "gop_s": ops / med / 1e6,
                       "ms_single_launch": one, "gop_s_single_launch": ops / one / 1e6,
                       "note": "latency-bound correctness config; mm_execute: 17 COMPUTE cuboids as one paco_mm_batch "
                               "launch, 4 REDUCEs fused into its epilogues; time is host-bound (plan walk)"}

    if 2 in only:  # cfg2: (min,+) 8192^3
        n = 8192
        a = torch.randint(0, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
        b = torch.randint(0, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
        a[torch.rand(n, n, device="cuda", generator=g) < 0.1] = 2**30
        b[torch.rand(n, n, device="cuda", generator=g) < 0.1] = 2**30
        c = torch.full((n, n), 2**30, device="cuda", dtype=torch.int32)
        med, best = timed(lambda: launch_mm(nat.SR_MINPLUS_SAT32, st, View.of(a), View.of(b), View.of(c)), args.reps)
        ops = 2 * n ** 3
        res["cfg2"] = {"ms": med, "top_s": ops / med / 1e9, "frac_alu_peak": ops / med / 1e9 / alu_peak}
        del a, b, c

    if 3 in only:  # cfg3: bf16 65536x256 @ 256x1024 -> fp32
        n, k, m = 65536, 256, 1024
        a = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
        b = torch.randn(k, m, device="cuda", generator=g).to(torch.bfloat16)
        c = torch.empty(n, m, device="cuda")
        av, bv, cv = View.of(a), View.of(b), View.of(c)
        reps = 20

        def run():
            for _ in range(reps):
                launch_mm(nat.SR_BF16_F32, st, av, bv, cv, overwrite=True)
        med, best = timed(run, 3)
        med /= reps
        byts = 2 * n * k + 2 * k * m + 4 * n * m
        res["cfg3"] = {"us": med * 1e3, "tflop_s": 2 * n * m * k / med / 1e9,
                       "gb_s_algorithmic": byts / med / 1e6, "frac_hbm": byts / med / 1e6 / HBM,
                       "alg_bytes": byts}
        del a, b, c

    if 4 in only:  # cfg4: (max,+) 16384^3 on one GPU, plus the p-way GPU-level plans on one GPU
        n = 16384
        a = torch.randint(-2**20, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
        b = torch.randint(-2**20, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
        c = torch.full((n, n), -2**30, device="cuda", dtype=torch.int32)
        med, best = timed(lambda: launch_mm(nat.SR_MAXPLUS_SAT32, st, View.of(a), View.of(b), View.of(c)),
                          max(2, args.reps // 2), warm=1)
        ops = 2 * n ** 3
        res["cfg4"] = {"ms": med, "top_s": ops / med / 1e9, "frac_alu_peak": ops / med / 1e9 / alu_peak}
        del a, b, c

    if 5 in only:  # cfg5: Strassen fp32 n=16384, 2 levels, 3xTF32 tcgen05 leaves
        n = 16384
        a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
        b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
        med, best = timed(lambda: S.strassen_seq(a, b, n, base=n // 4), 2, warm=1)
        alg = 49 * 2 * 4096 ** 3 + 18 * 8192 ** 2 + 7 * 18 * 4096 ** 2
        res["cfg5"] = {"ms": med, "tflop_s_algorithmic": alg / med / 1e9,
                       "tflop_s_classic_equivalent": 2 * n ** 3 / med / 1e9,
                       "frac_ffma_peak": alg / med / 1e9 / ffma_peak, "alg_flop": alg}
        # the leaves run 3xTF32 on the tensor pipe: whole-step tensor work vs the
        # TF32 dense peak (half the measured bf16 cuBLAS rate of MEASURED_PEAKS.json)
        tf32_peak = PEAKS.get("bf16_tflops", 2250.0) / 2
        mma = 3 * 49 * 2 * 4096 ** 3
        res["cfg5"].update({"tf32x3_mma_flop": mma, "tensor_tflop_s": mma / med / 1e9,
                            "tf32_peak_tflop_s": tf32_peak, "frac_tf32_tensor_peak": mma / med / 1e9 / tf32_peak,
                            "tf32_peak_source": "MEASURED_PEAKS.json bf16_tflops / 2" if "bf16_tflops" in PEAKS
                            else "nominal 2250 / 2"})
        del a, b
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

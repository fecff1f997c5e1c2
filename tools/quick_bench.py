"""Ad-hoc timing of paco_mm on one config (dev tool; bench.py is the contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

def run(sr, n, m, k, dtype, reps=5, pieces=None):
    g = torch.Generator(device="cuda").manual_seed(0)
    if dtype == torch.int32:
        A = torch.randint(0, 2**20, (n, k), device="cuda", dtype=torch.int32, generator=g)
        B = torch.randint(0, 2**20, (k, m), device="cuda", dtype=torch.int32, generator=g)
        C = torch.full((n, m), 2**30, device="cuda", dtype=torch.int32)
    else:
        A = torch.randn(n, k, device="cuda", generator=g).to(dtype)
        B = torch.randn(k, m, device="cuda", generator=g).to(dtype)
        C = torch.zeros(n, m, device="cuda", dtype=torch.float32 if dtype != torch.float64 else dtype)
    st = torch.cuda.current_stream()
    a, b, c = View.of(A), View.of(B), View.of(C)
    for _ in range(2):
        launch_mm(sr, st, a, b, c, pieces=pieces)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); launch_mm(sr, st, a, b, c, pieces=pieces); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    print(f"sr={sr} {n}x{m}x{k}: {t:.3f} ms  {2*n*m*k/t/1e9:.1f} Gop/s  (all: {[round(x,2) for x in ts]})", flush=True)
    return t

lib = nat.load()
for which, name in ((0, "viaddmnmx.u32"), (1, "viaddmnmx.s32"), (2, "ffma")):
    tpc = ctypes.c_double(); mhz = ctypes.c_double()
    nat.check(lib.paco_alu_probe(0, None, which, 20000, ctypes.byref(tpc), ctypes.byref(mhz)))
    print(f"alu probe {name}: {tpc.value:.2f} terms/clk/SM at {mhz.value:.0f} MHz -> {2*tpc.value*148*mhz.value/1e6:.1f} Top/s", flush=True)
args = sys.argv[1:]
run(nat.SR_MINPLUS_SAT32, 8192, 8192, 8192, torch.int32)
run(nat.SR_MAXPLUS_SAT32, 8192, 8192, 8192, torch.int32)
run(nat.SR_F32, 8192, 8192, 8192, torch.float32)
run(nat.SR_MINPLUS_SAT32, 4096, 4096, 4096, torch.int32)

"""Where cfg1's time goes (384x256x320 (+,x) int32 -> int64, PACO p=3).

Reports the GPU time of one `paco_mm` launch (CUDA graph of 100 launches,
so no host cost), the eager per-launch cost (100 back-to-back launches),
and `mm_execute` host wall time vs its GPU span.

    python tools/cfg1_latency.py
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm


def ev_time(fn, reps=100):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    g = torch.Generator(device="cuda").manual_seed(2011)
    a = torch.randint(-8, 9, (384, 256), device="cuda", dtype=torch.int32, generator=g)
    b = torch.randint(-8, 9, (256, 320), device="cuda", dtype=torch.int32, generator=g)
    c = torch.zeros(384, 320, device="cuda", dtype=torch.int64)
    av, bv, cv = View.of(a), View.of(b), View.of(c)
    out = {}
    for flags, name in ((0, "accumulate"), (nat.MM_OVERWRITE, "overwrite")):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            fn = lambda: launch_mm(nat.SR_INT_I32_I64, st, av, bv, cv, flags=flags)
            out[f"eager_ms_{name}"] = ev_time(fn)
            fn()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=st):
                for _ in range(100):
                    fn()
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            graph.replay()
            e1.record(st)
            e1.synchronize()
            out[f"graph_ms_{name}"] = e0.elapsed_time(e1) / 100
    ks, ctas = nat.cta_grid(nat.SR_INT_I32_I64, 384, 320, 256)
    out["cta_grid"] = {"ksplit": ks, "ctas": ctas, "tile_shape": nat.tile_shape(nat.SR_INT_I32_I64)}
    bm, bn, kq, _ = nat.tile_shape(nat.SR_INT_I32_I64)
    ku = -(-256 // kq)
    tiles = [(i, j) for i in range(-(-384 // bm)) for j in range(-(-320 // bn))]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for s in (1, 2, 4, 8, 16, 32):
            if s > ku:
                break
            pieces = [(i, j, p * ku // s, 1, 1, (p + 1) * ku // s - p * ku // s) for i, j in tiles for p in range(s)]
            fn = lambda: launch_mm(nat.SR_INT_I32_I64, st, av, bv, cv, pieces=pieces)
            fn()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=st):
                for _ in range(50):
                    fn()
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            graph.replay()
            e1.record(st)
            e1.synchronize()
            out[f"graph_ms_ksplit{s}"] = e0.elapsed_time(e1) / 50
    plan = M.mm_paco_partition(384, 320, 256, 3)
    for _ in range(3):
        M.mm_execute(plan, a, b, c, M.SEMIRING_INT)
    walls, gpus = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        rep = M.mm_execute(plan, a, b, c, M.SEMIRING_INT)
        walls.append((time.perf_counter() - t0) * 1e3)
        gpus.append(rep.gpu_ms)
    walls.sort()
    gpus.sort()
    out["mm_execute_wall_ms_median"] = walls[10]
    out["mm_execute_gpu_span_ms_median"] = gpus[10]
    print(out)


if __name__ == "__main__":
    main()

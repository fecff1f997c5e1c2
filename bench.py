"""Benchmark of the B200 PACO semiring-MM hot path (BASELINE.json's metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--cfg 2|3|4|5] [--configs 1,2,3,4,5|none]

Headline (``value``): cfg2, (min,+) saturating tropical MM n=m=k=8192
(BASELINE.json configs[1], the config the metric is quoted on).  One step =
one full C (+)= A (x) B over the 8192^3 iteration cuboid, inputs resident in
HBM: the GPU-level PACO plan (mm_one_piece_partition over N ranks,
matmul.py:250-300) gives each rank one cuboid; inside each rank one sm_100a
launch covers it with the tile-grid CTA plan; k-cut folds (N >= 5) are fused
into the kernels (upper-k ranks fold straight into the owner's C over CUDA
IPC / NVLink; --fold nccl uses NCCL MIN reductions instead).  The timed
region is bracketed by barrier + synchronize, timed with CUDA events and
max'ed over ranks.  A, B (256 MiB each) exceed the 126 MB L2: no flush needed.

``configs`` (N=1): every BASELINE config measured in the same run -- cfg1..cfg5
with ms, throughput, algorithmic ops/bytes, roofline fraction against a live
or driver-measured peak, launches and a clocks sample of its own timed region.

``e2e``: the same metric through the reference-facing API
``matmul.mm_seq(A, B, C, SEMIRING_MINPLUS_SAT)`` with NumPy arrays (the
reference's own calling convention; page-locked in place on first use): the
H2D of A, B, C and the D2H of C are inside the host-wall-clock timed region.  At N>1
``FusedDistributedMM.run_host`` from pinned host tensors.

``--impl reference`` times the reference's CPU algorithm (the NumPy port in
oracle/, process-sharded over every host core) on a bounded row sample of the
same config, plus one sample of the reference's threaded parallel mode.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "semiring MM Gop/s at 1/2/4/8 B200, % of roofline, vs CPU ref on host cores"
INF = 2**30
SM_COUNT = 148

WORKLOADS = {
    1: "cfg1: (+,x) int32 [-8,8] 384x256 . 256x320 -> int64, mm_paco_partition p=3 (BASELINE.json configs[0])",
    2: "cfg2: (min,+) saturating tropical MM n=m=k=8192, int32 [0,2^20) + 10% INF=2^30 (BASELINE.json configs[1])",
    3: "cfg3: (+,x) bf16 N(0,1) 65536x256 . 256x1024 -> fp32, tcgen05 (BASELINE.json configs[2])",
    4: "cfg4: (max,+) MM n=m=k=16384, int32 [-2^20,2^20) (BASELINE.json configs[3])",
    5: "cfg5: Strassen (+,x) fp32 U(-1,1) n=16384, 2 levels (49 leaves of 4096^3), tcgen05 leaves "
       "(BASELINE.json configs[4])",
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    """MEASURED_PEAKS.json (driver-written), else the profiling guide's stated fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "of measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "of fallback (B200_PROFILING.md: 6.65 TB/s, 1.59 PFLOP/s)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during a timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period: float = 0.1):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def ncu_traffic(name):
    """DRAM bytes per launch of a kernel from a committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        k = json.load(open(path))["kernels"][0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = sum(float(k[m]["value"]) * scale[k[m]["unit"]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return tot, os.path.relpath(path, ROOT)
    except Exception:
        return None, None


def alu_probe(device, which):
    """Issue rate of one term (0: VIADDMNMX.U32 min-plus, 1: VIADDMNMX.S32 max-plus), terms/clk/SM."""
    from paper_2011_01441_b200 import _native as nat

    tpc, mhz = ctypes.c_double(), ctypes.c_double()
    nat.check(nat.load().paco_alu_probe(device, None, which, 20000, ctypes.byref(tpc), ctypes.byref(mhz)))
    return tpc.value, mhz.value


def cpu_baseline(rows_per_proc=48, repeat=1):
    out = subprocess.run([sys.executable, "-m", "oracle.cpu_baseline", "--cfg", "2",
                          "--rows-per-proc", str(rows_per_proc), "--repeat", str(repeat)], cwd=ROOT,
                         capture_output=True, text=True, timeout=1800)
    if out.returncode != 0:
        return {"value": None, "unit": "Gop/s", "cores": None, "kind": "port",
                "sample": "failed: " + out.stderr.strip()[-200:]}
    return json.loads(out.stdout.strip().splitlines()[-1])


def workload_config(cfg):
    """The ``config`` object: identical in both arms for the same workload."""
    return {"workload": WORKLOADS[cfg],
            "inputs": f"numpy default_rng({1000 + cfg}) draws, A then B (SURVEY.md 8d)"}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm on the host cores.

    Each step is a bounded sample of cfg2 (full k and m, a slab of rows) run
    by the reference algorithm's NumPy port process-sharded over every host
    core; ``value`` is that sample's op count over its wall time.  Before the
    steps, one sample of the reference's shipped threaded mode
    (mm_execute(..., mode="parallel"), GIL-bound) is timed and reported."""
    if rank != 0:
        return
    from oracle import cpu_baseline as cb

    threaded = cb.measure_threaded(2, args.ref_threaded_rows)
    last = cpu_baseline(rows_per_proc=args.ref_rows, repeat=args.warmup + args.steps)
    vals = (last.get("values") or [last["value"]])[args.warmup:] or [last["value"]]
    value = statistics.median(vals)
    rows = args.ref_rows * last["cores"]
    sample_ops = 2.0 * rows * 8192 * 8192
    ms = sample_ops / (value * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gop/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded numpy default_rng(1002), BASELINE cfg2 distribution)",
        "config": workload_config(2),
        "step": f"one bounded sample per step: {rows} of the 8192 rows of A at full k and m "
                f"({sample_ops:.3e} ops, {ms / 1e3:.2f} s)",
        "cpu_baseline": {"value": value, "unit": "Gop/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"], "cpu_model": cb.cpu_model(),
                         "threaded_parallel_mode": threaded},
        "e2e": {"value": value, "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm: configs

def _events_time(fn, steps, warmup, st, per_step_calls=1):
    """CUDA-event time (ms) of `steps` calls of fn on stream st after `warmup` calls."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def _graph_time(launch, steps, warmup, st, dev, per_graph=20):
    """CUDA-event time (ms) per launch of ``launch(stream)`` captured ``per_graph``
    times into one CUDA graph, replayed on stream st after warm-up replays."""
    import torch

    cap = torch.cuda.Stream(dev)
    cap.wait_stream(st)
    launch(cap)  # per-stream library state (tile counters) is set up outside the capture
    cap.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        for _ in range(per_graph):
            launch(cap)
    st.wait_stream(cap)
    reps = max(1, -(-steps // per_graph))
    with torch.cuda.stream(st):
        for _ in range(max(1, -(-warmup // per_graph))):
            g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
        e1.synchronize()
    del g
    return e0.elapsed_time(e1) / (reps * per_graph)


def measure_config(cfg, dev, args, peaks, probes):
    """One BASELINE config on this GPU: dict for the line's ``configs``."""
    import numpy as np
    import torch

    from paper_2011_01441_b200 import _native as nat
    from paper_2011_01441_b200 import matmul as M
    from paper_2011_01441_b200 import strassen as S
    from paper_2011_01441_b200.device import View
    from paper_2011_01441_b200.mm import launch_mm

    st = torch.cuda.current_stream(dev)
    rng = np.random.default_rng(1000 + cfg)
    out = {"workload": WORKLOADS[cfg]}
    if cfg == 1:
        A = rng.integers(-8, 9, (384, 256), dtype=np.int32)
        B = rng.integers(-8, 9, (256, 320), dtype=np.int32)
        a, b = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
        c = torch.zeros(384, 320, dtype=torch.int64, device=dev)
        plan = M.mm_paco_partition(384, 320, 256, 3)
        steps, warmup = max(100, args.steps * 5), max(3, args.warmup)
        with ClockSampler(dev, 0.02) as clk:
            ms = _events_time(lambda: M.mm_execute(plan, a, b, c, M.SEMIRING_INT), steps, warmup, st)
        ops = 2.0 * 384 * 320 * 256
        out.update(ms=ms, value=ops / ms / 1e6, unit="Gop/s", ops_per_step=ops, steps=steps, warmup=warmup,
                   algorithmic_bytes=1703936, gpu_launches_per_step=1,
                   step="mm_execute(mm_paco_partition(384,320,256,3), device int32 A/B, int64 C, SEMIRING_INT): "
                        "17 COMPUTE cuboids as one paco_mm_batch launch, 4 REDUCEs fused into its epilogues; "
                        "includes the host-side plan walk",
                   roofline={"bound": "latency", "note": "correctness config (0.06 Gop per step): no roofline "
                                                          "claim (SURVEY.md 8d)"},
                   clocks=clk.summary())
        return out
    if cfg in (2, 4):
        n = 8192 if cfg == 2 else 16384
        if cfg == 2:
            A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
            A[rng.random(A.shape) < 0.10] = INF
            B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
            B[rng.random(B.shape) < 0.10] = INF
        else:
            A = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
            B = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
        a, b = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
        del A, B
        kid = nat.SR_MINPLUS_SAT32 if cfg == 2 else nat.SR_MAXPLUS_SAT32
        c = torch.full((n, n), INF if cfg == 2 else -INF, dtype=torch.int32, device=dev)
        av, bv, cv = View.of(a), View.of(b), View.of(c)
        steps = args.steps if cfg == 2 else max(3, min(args.steps, 6))
        warmup = max(3, args.warmup) if cfg == 2 else 3
        with ClockSampler(dev) as clk:
            ms = _events_time(lambda: launch_mm(kid, st, av, bv, cv), steps, warmup, st)
        ops = 2.0 * n ** 3
        tpc, probe_mhz = probes[0 if cfg == 2 else 1]
        peak = 2 * tpc * SM_COUNT * 1965.0 / 1e6
        achieved = ops / ms / 1e9
        clocks = clk.summary()
        traffic, src = ncu_traffic("r2_minplus_tma_ncu.json" if cfg == 2 else "r2_maxplus_tma_ncu.json")
        ks, ctas = nat.cta_grid(kid, n, n, n)
        out.update(ms=ms, value=ops / ms / 1e6, unit="Gop/s", ops_per_step=ops, steps=steps, warmup=warmup,
                   algorithmic_bytes=3 * n * n * 4, gpu_launches_per_step=1,
                   step=f"one paco_mm launch (simt_mm_kernel, {ctas} CTAs: 128x128 C tiles, k split {ks} way(s) "
                        "+ tail split), device-resident operands",
                   l2=f"inputs 2 x {n * n * 4 >> 20} MiB > 126 MB L2 (no flush)",
                   roofline={"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Top/s",
                             "frac": achieved / peak,
                             "peak_source": (f"live VIADDMNMX.{'U32' if cfg == 2 else 'S32'} probe: {tpc:.2f} "
                                             f"terms/clk/SM x 2 op x 148 SM x 1965 MHz max clock (probe ran at "
                                             f"{probe_mhz:.0f} MHz)"),
                             "peak_at_run_clock": (2 * tpc * SM_COUNT * clocks["sm_mhz"] / 1e6
                                                   if clocks.get("sm_mhz") else None),
                             "traffic": traffic, "traffic_source": src, "algorithmic_bytes": 3 * n * n * 4},
                   clocks=clocks)
        if cfg == 2:
            # the north star's second PACO level as the CTA plan (MM-1-Piece over 148 x 2 x 4 workers)
            # beside the default tile grid, same launches, same inputs
            paco_ms = _events_time(lambda: launch_mm(kid, st, av, bv, cv, flags=nat.MM_PACO_PLAN), 3, 1, st)
            out["cta_plan_compare"] = {
                "tile_grid_ms": ms, "paco_cuboid_plan_ms": paco_ms,
                "paco_cuboid_plan": "PACO_MM_PACO_PLAN: paco_plan_cta's MM-1-Piece over the (128, 128, 4) unit grid "
                                    "for p = 1184 workers (DESIGN.md section 5)"}
        out["_tensors"] = (a, b, c)
        return out
    if cfg == 3:
        n, k, m = 65536, 256, 1024
        A = rng.standard_normal((n, k), dtype=np.float32)
        B = rng.standard_normal((k, m), dtype=np.float32)
        a = torch.from_numpy(A).to(dev).to(torch.bfloat16)
        b = torch.from_numpy(B).to(dev).to(torch.bfloat16)
        c = torch.empty(n, m, dtype=torch.float32, device=dev)
        av, bv, cv = View.of(a), View.of(b), View.of(c)
        steps, warmup = max(200, args.steps * 10), max(10, args.warmup)
        # timed as CUDA-graph replays of 20 captured launches each (the launch-bound
        # loop in a graph: ~2.3 us less per launch than direct launches, kept as ms_direct)
        with ClockSampler(dev, 0.02) as clk:
            ms = _graph_time(lambda s_: launch_mm(nat.SR_BF16_F32, s_, av, bv, cv, overwrite=True), steps, warmup,
                             st, dev)
            ms_direct = _events_time(lambda: launch_mm(nat.SR_BF16_F32, st, av, bv, cv, overwrite=True), steps,
                                     warmup, st)
        # the same launches one at a time after a 512 MiB L2 flush each (cold L2, event pair per launch)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        cold = []
        for i in range(20):
            flush.fill_(i & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            launch_mm(nat.SR_BF16_F32, st, av, bv, cv, overwrite=True)
            e1.record(st)
            e1.synchronize()
            cold.append(e0.elapsed_time(e1))
        del flush
        byts = 2 * n * k + 2 * k * m + 4 * n * m
        flop = 2.0 * n * m * k
        achieved = byts / ms / 1e6
        traffic, src = ncu_traffic("r2_bf16_ncu.json")
        out.update(ms=ms, value=flop / ms / 1e6, unit="Gop/s", ops_per_step=flop, steps=steps, warmup=warmup,
                   algorithmic_bytes=byts, gpu_launches_per_step=1,
                   ms_direct=ms_direct, ms_l2_flushed=statistics.median(cold),
                   step="one paco_mm launch (tc_gemm_kernel<KindBF16Res>: persistent tcgen05, resident B), "
                        "C overwritten (fp32, not read); steps replayed from a CUDA graph of 20 launches "
                        "(ms_direct: the same launches issued one by one)",
                   l2="back-to-back launches; working set 302 MB > 126 MB L2 (the 268 MB fp32 C write "
                      "evicts A); ms_l2_flushed: each launch alone after a 512 MiB flush",
                   roofline={"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": achieved / peaks["hbm_gbs"],
                             "frac_direct": byts / ms_direct / 1e6 / peaks["hbm_gbs"],
                             "frac_l2_flushed": byts / statistics.median(cold) / 1e6 / peaks["hbm_gbs"],
                             "peak_source": f"hbm_gbs {peaks['source']}",
                             "traffic": traffic, "traffic_source": src, "algorithmic_bytes": byts},
                   clocks=clk.summary())
        return out
    if cfg == 5:
        n = 16384
        A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        a, b = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
        del A, B
        steps, warmup = max(3, min(args.steps, 10)), 3
        fn = lambda: S.strassen_seq(a, b, n, base=n // 4)  # noqa: E731
        with ClockSampler(dev) as clk:
            ms = _events_time(fn, steps, warmup, st)
        # live per-kernel timing of the same step (event pair around every launch; a separate pass)
        with nat.kernel_timing() as kt:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            fam = {name: kt.read(f) for name, f in (("tc_gemm", nat.KT_TC_GEMM), ("tf32_split", nat.KT_TF32_SPLIT),
                                                    ("lincomb", nat.KT_LINCOMB),
                                                    ("elementwise", nat.KT_ELEMENTWISE))}
        per_step = {k_: {"ms": v[0] / 3, "launches": v[1] // 3} for k_, v in fam.items()}
        alg = 49 * 2 * 4096 ** 3 + 18 * 8192 ** 2 + 7 * 18 * 4096 ** 2
        lw = leaf_work(S, peaks)
        mma = 49 * lw["per_product"]
        leaf_ms = per_step["tc_gemm"]["ms"]
        leaf_launch_ms = leaf_ms / max(1, per_step["tc_gemm"]["launches"])
        leaf_flop = mma / max(1, per_step["tc_gemm"]["launches"])   # one launch = 7 products of 4096^3
        achieved = leaf_flop / leaf_launch_ms / 1e9
        traffic, src = ncu_traffic(lw["ncu"])
        out.update(ms=ms, value=alg / ms / 1e6, unit="Gop/s", ops_per_step=alg, steps=steps, warmup=warmup,
                   classic_equivalent_gop_s=2.0 * n ** 3 / ms / 1e6,
                   gpu_launches_per_step=sum(v["launches"] for v in per_step.values()),
                   kernels_per_step=per_step, leaf_format=lw["format"],
                   step="strassen_seq(A, B, 16384, base=4096): 2 Strassen levels, 49 leaf products of 4096^3 on CTA "
                        "pairs (tcgen05 cta_group::2; 7 batched launches), C combination fused into the leaf epilogues",
                   l2="A, B 1 GiB each > 126 MB L2 (no flush)",
                   roofline={"bound": "tensor", "kernel": "tc_pair_kernel (Strassen leaves on CTA pairs)",
                             "achieved": achieved, "peak": lw["peak"], "unit": lw["unit"],
                             "frac": achieved / lw["peak"], "frac_burst": achieved / lw["peak_burst"],
                             "achieved_note": ("tensor work of one launch (7 products of 4096^3: " + lw["note"] +
                                               ") / its average CUDA-event duration inside the step"),
                             "step_frac": mma / ms / 1e9 / lw["peak"],
                             "step_note": "whole step: 49 leaf products' tensor work / step time",
                             "peak_source": lw["peak_source"],
                             "traffic": traffic, "traffic_source": src},
                   clocks=clk.summary())
        return out
    raise ValueError(cfg)


def leaf_work(S, peaks):
    """Tensor work of one cfg5 leaf product (4096^3) in the leaf format the library
    runs, and the peak it is held to.  The leaf launches run inside a ~20 ms step
    repeated back to back, so the denominator is the SUSTAINED bf16 figure of
    MEASURED_PEAKS.json (B200_PROFILING: burst for a kernel timed alone, sustained
    for one inside a long step); frac_burst is reported beside it."""
    p3 = 2 * 4096 ** 3
    if S.LEAF_BF16X3:
        return {"per_product": 3 * p3, "unit": "TFLOP/s (bf16)", "peak": peaks["bf16_tflops_sustained"],
                "peak_burst": peaks["bf16_tflops"], "ncu": "r2_bf16x3_ncu.json",
                "note": "3 bf16 products (hi*hi, hi*lo, lo*hi) x 2 x 4096^3 each",
                "format": ("bf16x3: operands as bf16 hi/lo planes (one paco_lincomb_split pass per node side), "
                           "hi*hi + hi*lo + lo*hi on kind::f16, fp32 accumulation"),
                "peak_source": (f"bf16_tflops_sustained {peaks['source']} (kernel inside a long step; "
                                f"burst {peaks['bf16_tflops']:.1f} gives frac_burst)")}
    b2 = S.TF32B2
    return {"per_product": (2 if b2 else 3) * p3, "unit": "TFLOP/s (tf32-equivalent)",
            "peak": peaks["bf16_tflops_sustained"] / 2, "peak_burst": peaks["bf16_tflops"] / 2,
            "ncu": "r2_tf32b2_raw_ncu.json",
            "note": ("2" if b2 else "3") + " tf32-equivalent products x 2 x 4096^3 each (a bf16 MMA counts half)",
            "format": ("tf32 + 2 x bf16 split products, fp32 accumulation" if b2
                       else "3xTF32 split products, fp32 accumulation"),
            "peak_source": f"TF32 dense = bf16_tflops_sustained / 2 {peaks['source']}"}


def e2e_numpy_cfg2(dev, steps):
    """cfg2 end to end through matmul.mm_seq with pageable NumPy A, B, C (host wall clock)."""
    import numpy as np
    import torch

    from paper_2011_01441_b200 import matmul as M

    rng = np.random.default_rng(1002)
    n = 8192
    A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
    A[rng.random(A.shape) < 0.10] = INF
    B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
    B[rng.random(B.shape) < 0.10] = INF
    C = np.full((n, n), INF, np.int32)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)  # first call: page-locks A, B, C once (paco_host_register)
    first_ms = (time.perf_counter() - t0) * 1e3
    times = []
    for _ in range(steps):
        C.fill(INF)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
        times.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(times)
    return {"value": 2.0 * n ** 3 / (ms * 1e-3) / 1e9, "unit": "Gop/s", "ms_per_step": ms,
            "ms_all": times, "first_call_ms": first_ms, "h2d_bytes_per_step": 3 * n * n * 4,
            "d2h_bytes_per_step": n * n * 4,
            "api": "paper_2011_01441_b200.matmul.mm_seq(A, B, C, SEMIRING_MINPLUS_SAT) with NumPy int32 arrays: "
                   "page-locked in place on first use (paco_host_register, first_call_ms), then every call DMAs A, "
                   "B, C up and C back through the k-phased H2D/compute/D2H pipeline; host wall clock"}


def e2e_pinned_cfg2(dev, st, A_h, B_h, steps):
    import torch

    from paper_2011_01441_b200 import matmul as M

    n = 8192
    C_h = torch.full((n, n), INF, dtype=torch.int32).pin_memory()
    M.mm_seq(A_h, B_h, C_h, M.SEMIRING_MINPLUS_SAT)  # warm
    torch.cuda.synchronize(dev)
    t = []
    for _ in range(steps):
        C_h.fill_(INF)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        M.mm_seq(A_h, B_h, C_h, M.SEMIRING_MINPLUS_SAT)
        t.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(t)
    return {"value": 2.0 * n ** 3 / (ms * 1e-3) / 1e9, "unit": "Gop/s", "ms_per_step": ms,
            "api": "matmul.mm_seq with pinned torch host tensors; host wall clock"}


# ----------------------------------------------------------------------------- our arm: main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=2, choices=[2, 3, 4, 5],
                    help="headline config at N>1 (GPU-level PACO plan of that BASELINE config)")
    ap.add_argument("--configs", default="1,2,3,4,5",
                    help="N=1: BASELINE configs measured into the line's `configs` ('none' to skip)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-rows", type=int, default=24, help="rows of A per host process (reference arm)")
    ap.add_argument("--ref-threaded-rows", type=int, default=32, help="rows of A for the threaded-mode sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fold", default="fused", choices=["fused", "nccl"],
                    help="N>1: k-cut folds fused into the kernels over IPC, or NCCL reductions")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2011_01441_b200 import _native as nat

    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL needs one GPU per rank; with more ranks than GPUs (a test box) use gloo
        backend = os.environ.get("PACO_BENCH_BACKEND",
                                 "nccl" if torch.cuda.device_count() >= world else "gloo")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)

    peaks = load_peaks()
    probes = {0: alu_probe(dev, 0), 1: alu_probe(dev, 1)}
    cfg = 2 if world == 1 else args.cfg
    st = torch.cuda.current_stream(dev)
    configs = {}
    wanted = [] if args.configs == "none" or world > 1 else [int(x) for x in args.configs.split(",") if x]

    if world == 1:
        # the headline IS configs.cfg2: measured once, with the contract's K/W and barrier-free timing
        res2 = measure_config(2, dev, args, peaks, probes)
        a, b, c = res2.pop("_tensors")
        ms = res2["ms"]
        n = 8192
        ops_per_step = 2.0 * n ** 3
        ks, ctas = nat.cta_grid(nat.SR_MINPLUS_SAT32, n, n, n)
        plan_desc = (f"1 GPU, CTA-level tile grid: {ctas} CTAs of one 128x128 C tile, k split {ks} way(s) "
                     "(cost-model choice over the PACO cuboid plan, DESIGN.md section 5)")
        launches_per_step = 1
        clocks = res2["clocks"]
        roofline = res2["roofline"]
        A_h, B_h = a.cpu().pin_memory(), b.cpu().pin_memory()
        del a, b, c
        torch.cuda.empty_cache()
        dtype, l2 = "u32", f"inputs 2 x {n * n * 4 >> 20} MiB > 126 MB L2 (no flush)"
    else:
        mg = MultiGPU(cfg, world, rank, dev, args, peaks, probes)
        ops_per_step, plan_desc, launches_per_step, dtype, l2 = (mg.ops_per_step, mg.plan_desc,
                                                                 mg.launches_per_step, mg.dtype, mg.l2)

        def barrier():
            dist.barrier()
            torch.cuda.synchronize(dev)

        for _ in range(args.warmup):
            mg.step()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(dev) as clk:
            barrier()
            e0.record(st)
            for _ in range(args.steps):
                mg.step()
            e1.record(st)
            barrier()
        t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item()) / args.steps
        clocks = clk.summary()
        roofline = mg.roofline(ms)

    value = ops_per_step / (ms * 1e-3) / 1e9  # whole-job Gop/s

    # e2e through the public API from host memory
    if world == 1:
        e2e = e2e_numpy_cfg2(dev, args.e2e_steps)
        e2e["pinned_torch"] = e2e_pinned_cfg2(dev, st, A_h, B_h, args.e2e_steps)
    else:
        e2e = mg.e2e(args.e2e_steps)

    if world == 1:
        configs["cfg2"] = res2
        for c_ in wanted:
            if c_ == 2:
                continue
            torch.cuda.empty_cache()
            r = measure_config(c_, dev, args, peaks, probes)
            r.pop("_tensors", None)
            configs[f"cfg{c_}"] = r
        configs = {k_: configs[k_] for k_ in sorted(configs)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gop/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype,
            "data": f"synthetic (seeded numpy default_rng({1000 + cfg}), BASELINE cfg{cfg} distribution)",
            "config": workload_config(cfg),
            "plan": plan_desc,
            "l2": l2,
            "ops_per_step": ops_per_step,
            "roofline": roofline,
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
        }
        if configs:
            line["configs"] = configs
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class MultiGPU:
    """One rank's share of a BASELINE config at N > 1 GPUs (one process per GPU).

    cfg2 / cfg4: GPU-level MM-1-Piece (k-cut folds fused into the kernels over
    IPC, or NCCL reductions with --fold nccl).  cfg3: MM-1-Piece's n-only cuts
    of the skinny shape, B replicated, every rank's block a sole-writer tcgen05
    launch (no exchange).  cfg5: DistributedStrassen (PACO-balanced nodes and
    split leftover leaves, one NCCL reduce-scatter of the signed partials)."""

    def __init__(self, cfg, world, rank, dev, args, peaks, probes):
        import numpy as np
        import torch

        from paper_2011_01441_b200 import _native as nat
        from paper_2011_01441_b200 import matmul as M
        from paper_2011_01441_b200 import strassen as S
        from paper_2011_01441_b200.distributed import (CudaOps, CudaStrassenOps, DistributedMM,
                                                       DistributedStrassen, FusedDistributedMM)

        self.cfg, self.world, self.rank, self.dev, self.peaks = cfg, world, rank, dev, peaks
        self.torch, self.nat = torch, nat
        rng = np.random.default_rng(1000 + cfg)
        st = torch.cuda.current_stream(dev)
        self.l2 = "operands > 126 MB L2 (no flush)"
        if cfg in (2, 4):
            n = 8192 if cfg == 2 else 16384
            if cfg == 2:
                A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
                A[rng.random(A.shape) < 0.10] = INF
                B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
                B[rng.random(B.shape) < 0.10] = INF
            else:
                A = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
                B = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
            sr = M.SEMIRING_MINPLUS_SAT if cfg == 2 else M.SEMIRING_MAXPLUS
            kid = nat.SR_MINPLUS_SAT32 if cfg == 2 else nat.SR_MAXPLUS_SAT32
            self.A_h, self.B_h = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
            self.A, self.B = self.A_h.to(dev), self.B_h.to(dev)
            self.ops_per_step = 2.0 * n ** 3
            self.dtype = "u32" if cfg == 2 else "s32"
            self.l2 = f"inputs 2 x {n * n * 4 >> 20} MiB > 126 MB L2 (no flush)"
            self.tpc = probes[0 if cfg == 2 else 1][0]
            plan = M.mm_one_piece_partition(n, n, n, world, quantum=nat.tile_shape(kid)[:3])
            nred = sum(1 for t in plan.tasks if t.kind == "reduce")
            if args.fold == "fused":
                self.ex = FusedDistributedMM(plan, sr, kid, dev)
                self.step = lambda: self.ex.run(self.A, self.B)
                self.launches_per_step = len(self.ex.fill_rects) + len(self.ex.launches) + len(self.ex.incoming)
                how = ("staged: local temporary -> one NVLink copy into the owner's staging slot -> owner fold"
                       if self.ex.fold_style == "stage" else
                       f"{'TMA bulk' if self.ex.remote_bulk else 'element'} system-scope atomics into the owner's "
                       "C over NVLink")
                sync = "NCCL 1-element all-reduce (stream-ordered, no host sync)" if self.ex._nccl else \
                    "host barrier (gloo)"
                self.plan_desc = (f"{world} GPUs, GPU-level mm_one_piece_partition(p={world}, cuts on 128-row/column "
                                  f"tile multiples); its {nred} k-cut folds need no REDUCE temporaries or NCCL "
                                  f"reduction: local ones are fused into the kernels' epilogues, remote ones {how} "
                                  f"(CUDA IPC); fold handshake: {sync if self.ex.exchange else 'none (no k cut)'}; "
                                  "tile-grid CTA plan inside each rank")
                if self.ex.fold_probe_ms:
                    self.plan_desc += ("; fold style chosen by a start-up timing probe (1024^3 block, [fused, "
                                       f"staged] ms per rank: {[[round(x, 3) for x in t] for t in self.ex.fold_probe_ms]})")
            else:
                self.ex = DistributedMM(plan, sr, CudaOps(sr, kid, st))
                self.C = torch.empty((n, n), dtype=torch.int32, device=dev)
                mine = sum(1 for t in plan.tasks if t.kind == "reduce" and rank in t.workers())
                self.step = lambda: self.ex.run(self.A, self.B, self.C)
                self.launches_per_step = 2 + len(self.ex.temp_ids) + 3 * mine + len(self.ex.mine)
                self.plan_desc = (f"{world} GPUs, GPU-level mm_one_piece_partition(p={world}) ({nred} k-cut NCCL "
                                  f"{'MIN' if cfg == 2 else 'MAX'} folds), tile-grid CTA plan inside each rank")
        elif cfg == 3:
            n, k, m = 65536, 256, 1024
            A = rng.standard_normal((n, k), dtype=np.float32)
            B = rng.standard_normal((k, m), dtype=np.float32)
            self.A_h = torch.from_numpy(A).to(torch.bfloat16).pin_memory()
            self.B_h = torch.from_numpy(B).to(torch.bfloat16).pin_memory()
            self.A, self.B = self.A_h.to(dev), self.B_h.to(dev)
            plan = M.mm_one_piece_partition(n, m, k, world, quantum=nat.tile_shape(nat.SR_BF16_F32)[:3])
            self.ex = FusedDistributedMM(plan, M.SEMIRING_BF16, nat.SR_BF16_F32, dev)
            self.step = lambda: self.ex.run(self.A, self.B)
            self.launches_per_step = len(self.ex.fill_rects) + len(self.ex.launches)
            self.ops_per_step = 2.0 * n * m * k
            self.dtype = "bf16"
            rows = sum(r[2] for r in self.ex.owned)
            self.bytes_rank = 2 * rows * k + 2 * k * m + 4 * rows * m
            self.plan_desc = (f"{world} GPUs, mm_one_piece_partition(65536, 1024, 256, p={world}): n-only cuts, B "
                              f"replicated, each rank's {rows}-row block one sole-writer tcgen05 launch (C stored "
                              "once, no fill, no exchange)")
        elif cfg == 5:
            n = 16384
            A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
            B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
            self.A_h, self.B_h = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
            self.A, self.B = self.A_h.to(dev), self.B_h.to(dev)
            plan = S.strassen_paco_partition(n, world, base=n // 4, split_leftover=True)
            self.ex = DistributedStrassen(plan, CudaStrassenOps(torch.float32))
            self.step = lambda: self.ex.run(self.A, self.B)
            self.launches_per_step = None
            self.ops_per_step = 49 * 2 * 4096 ** 3 + 18 * 8192 ** 2 + 7 * 18 * 4096 ** 2
            self.dtype = "f32 (bf16x3 leaves)" if S.LEAF_BF16X3 else "f32 (tf32 + 2 x bf16 leaves)"
            self.plan_desc = (f"{world} GPUs, strassen_paco_partition(16384, p={world}, base=4096, split_leftover): "
                              f"{len(self.ex.nodes)} node(s) + {len(self.ex.pieces)} leaf piece(s) on this rank; "
                              "signed partial C folded by the leaf epilogues, then one NCCL reduce-scatter")
            with nat.kernel_timing() as kt:
                self.step()
                torch.cuda.synchronize(dev)
                self.launches_per_step = sum(kt.read(f)[1] for f in range(5))
        else:
            raise SystemExit(f"--cfg {cfg}: no multi-GPU bench for this config")

    def roofline(self, ms):
        per_gpu = self.ops_per_step / self.world / (ms * 1e-3)
        if self.cfg in (2, 4):
            peak = 2 * self.tpc * SM_COUNT * 1965.0 / 1e6
            return {"bound": "alu", "achieved": per_gpu / 1e12, "peak": peak, "unit": "Top/s",
                    "frac": per_gpu / 1e12 / peak, "per": "GPU (whole-job Top/s / N)",
                    "peak_source": f"live VIADDMNMX probe: {self.tpc:.2f} terms/clk/SM x 2 x 148 x 1965 MHz"}
        if self.cfg == 3:
            gbs = self.bytes_rank / (ms * 1e-3) / 1e9
            return {"bound": "hbm", "achieved": gbs, "peak": self.peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / self.peaks["hbm_gbs"], "per": "GPU (rank 0's algorithmic bytes / step time)",
                    "peak_source": f"hbm_gbs {self.peaks['source']}"}
        from paper_2011_01441_b200 import strassen as S
        lw = leaf_work(S, self.peaks)
        mma = 49 * lw["per_product"] / self.world
        tf = mma / (ms * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": tf, "peak": lw["peak"], "unit": lw["unit"],
                "frac": tf / lw["peak"], "frac_burst": tf / lw["peak_burst"],
                "per": "GPU (leaf tensor work / N / step time, reduce-scatter included)",
                "peak_source": lw["peak_source"]}

    def e2e(self, steps):
        """The same step from pinned host operands, host wall clock, max over ranks."""
        import torch
        import torch.distributed as dist

        torch_ = self.torch
        dev = self.dev
        if self.cfg in (2, 3, 4) and hasattr(self.ex, "run_host"):
            C_h = torch_.empty((self.ex.n, self.ex.m), dtype=self.ex.tdtype).pin_memory()
            fn = lambda: self.ex.run_host(self.A_h, self.B_h, C_h)  # noqa: E731
            api = "paper_2011_01441_b200.distributed.FusedDistributedMM.run_host (pinned host tensors)"
        elif self.cfg == 5:
            rows = self.ex.rows
            C_h = torch_.empty((rows, self.ex.size), dtype=torch_.float32).pin_memory()

            def fn():
                self.A.copy_(self.A_h, non_blocking=True)
                self.B.copy_(self.B_h, non_blocking=True)
                slab = self.ex.run(self.A, self.B)
                C_h.copy_(slab, non_blocking=True)
                torch_.cuda.synchronize(dev)
                n = self.A_h.shape[0]
                return (2 * n * n * 4, rows * self.ex.size * 4)
            api = ("paper_2011_01441_b200.distributed.DistributedStrassen.run with pinned A/B uploaded and the rank's "
                   "C row slab downloaded every step")
        else:
            return None
        fn()  # warm
        t_e2e, nbytes = [], (0, 0)
        for _ in range(steps):
            dist.barrier()
            torch_.cuda.synchronize(dev)
            t0 = time.perf_counter()
            nbytes = fn()
            torch_.cuda.synchronize(dev)
            t = torch_.tensor([(time.perf_counter() - t0) * 1e3], device=dev, dtype=torch_.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e.append(float(t.item()))
        tot = torch_.tensor(list(nbytes), device=dev, dtype=torch_.float64)
        dist.all_reduce(tot)
        ms = statistics.median(t_e2e)
        return {"value": self.ops_per_step / (ms * 1e-3) / 1e9, "unit": "Gop/s", "ms_per_step": ms,
                "h2d_bytes_per_step": int(tot[0].item()), "d2h_bytes_per_step": int(tot[1].item()),
                "bytes": "summed over ranks; time = max over ranks (host wall clock)", "api": api}


if __name__ == "__main__":
    main()

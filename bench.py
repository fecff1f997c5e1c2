"""Headline benchmark: (min,+) saturating tropical MM, n=m=k=8192 (BASELINE cfg2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full C (+)= A (x) B over the 8192^3 iteration cuboid, inputs
resident in HBM: the GPU-level PACO plan (mm_one_piece_partition over N ranks,
matmul.py:250-300) gives each rank one cuboid; inside each rank one sm_100a
launch covers it with the tile-grid CTA plan (one CTA per 128x128 C tile, k split
by the cost model); k-cut folds (N >= 5) are fused into the kernels (upper-k
ranks fold straight into the owner's C over CUDA IPC / NVLink; --fold nccl uses
NCCL MIN reductions instead).  The timed region
is bracketed by barrier + synchronize, timed with CUDA events and max'ed over
ranks.  A, B (256 MiB each) exceed the 126 MB L2, so no flush is needed.

``e2e`` runs the same metric through the public API (``matmul.mm_seq``; at N>1
``FusedDistributedMM.run_host``) from pinned HOST buffers: H2D of the operands
(and C at N=1) and D2H of C inside the timed region.

``--impl reference`` times the reference's CPU algorithm (the NumPy port in
oracle/, process-sharded over every host core) on a bounded row sample of the
same config.
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
N = 8192
INF = 2**30
OPS_PER_STEP = 2.0 * N * N * N
ALG_BYTES = 3 * N * N * 4  # A, B read once, C written once (int32)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
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
            self._stop.wait(0.2)

    def __enter__(self):
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_inputs(device):
    """cfg2 inputs: default_rng(1002), A then B, uniform [0, 2^20) with 10% INF."""
    import numpy as np
    import torch

    rng = np.random.default_rng(1002)
    A = rng.integers(0, 2**20, (N, N), dtype=np.int32)
    A[rng.random(A.shape) < 0.10] = INF
    B = rng.integers(0, 2**20, (N, N), dtype=np.int32)
    B[rng.random(B.shape) < 0.10] = INF
    A_h = torch.from_numpy(A).pin_memory()
    B_h = torch.from_numpy(B).pin_memory()
    return A_h, B_h


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "r1_minplus_ncu.json")
    try:
        k = json.load(open(path))["kernels"][0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = sum(float(k[m]["value"]) * scale[k[m]["unit"]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return tot, os.path.relpath(path, ROOT)
    except Exception:
        return None, None


def alu_peak(device):
    """VIADDMNMX.U32 issue rate measured live (terms/clk/SM) -> Top/s at a given clock."""
    from paper_2011_01441_b200 import _native as nat

    tpc, mhz = ctypes.c_double(), ctypes.c_double()
    nat.check(nat.load().paco_alu_probe(device, None, 0, 20000, ctypes.byref(tpc), ctypes.byref(mhz)))
    return tpc.value, mhz.value


def cpu_baseline(rows_per_proc=48, repeat=1):
    out = subprocess.run([sys.executable, "-m", "oracle.cpu_baseline", "--cfg", "2",
                          "--rows-per-proc", str(rows_per_proc), "--repeat", str(repeat)], cwd=ROOT,
                         capture_output=True, text=True, timeout=1800)
    if out.returncode != 0:
        return {"value": None, "unit": "Gop/s", "cores": None, "kind": "port",
                "sample": "failed: " + out.stderr.strip()[-200:]}
    return json.loads(out.stdout.strip().splitlines()[-1])


def run_reference(args, rank, world):
    """--impl reference: the reference CPU algorithm on the host cores."""
    if rank != 0:
        return
    last = cpu_baseline(rows_per_proc=args.ref_rows, repeat=args.warmup + args.steps)
    vals = (last.get("values") or [last["value"]])[args.warmup:] or [last["value"]]
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gop/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": OPS_PER_STEP / (value * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded, BASELINE cfg2 distribution)",
        "config": {"workload": "cfg2: (min,+) saturating MM n=m=k=8192, int32 [0,2^20) + 10% INF=2^30",
                   "sample_per_step": last["sample"]},
        "cpu_baseline": {"value": value, "unit": "Gop/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-rows", type=int, default=48, help="rows of A per host process (reference arm)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fold", default="fused", choices=["fused", "nccl"],
                    help="N>1: k-cut folds fused into the kernels over IPC, or NCCL reductions")
    args = ap.parse_args()

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2011_01441_b200 import _native as nat
    from paper_2011_01441_b200 import matmul as M
    from paper_2011_01441_b200.device import View
    from paper_2011_01441_b200.distributed import CudaOps, DistributedMM, FusedDistributedMM
    from paper_2011_01441_b200.mm import launch_mm

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

    A_h, B_h = make_inputs(dev)
    A = A_h.to(dev)
    B = B_h.to(dev)
    sr = M.SEMIRING_MINPLUS_SAT
    kid = nat.SR_MINPLUS_SAT32
    st = torch.cuda.current_stream(dev)

    if world == 1:
        C = torch.full((N, N), INF, dtype=torch.int32, device=dev)
        a, b, c = View.of(A), View.of(B), View.of(C)

        def step():
            launch_mm(kid, st, a, b, c)
        launches_per_step = 1
        ks, ctas = nat.cta_grid(kid, N, N, N)
        plan_desc = (f"1 GPU, CTA-level tile grid: {ctas} CTAs of one 128x128 C tile, k split {ks} way(s) "
                     "(cost-model choice over the PACO cuboid plan, DESIGN.md section 5)")
    elif args.fold == "fused":
        plan = M.mm_one_piece_partition(N, N, N, world, quantum=nat.tile_shape(kid)[:3])
        ex = FusedDistributedMM(plan, sr, kid, dev)
        nred = sum(1 for t in plan.tasks if t.kind == "reduce")

        def step():
            ex.run(A, B)
        launches_per_step = len(ex.owned) + len(ex.launches) + len(ex.incoming)
        how = ("staged: local temporary -> one NVLink copy into the owner's staging slot -> owner fold"
               if ex.fold_style == "stage" else
               f"{'TMA bulk' if ex.remote_bulk else 'element'} atomics into the owner's C over NVLink")
        plan_desc = (f"{world} GPUs, GPU-level mm_one_piece_partition(p={world}, cuts on 128-row/column tile "
                     f"multiples); its {nred} k-cut folds "
                     f"need no REDUCE temporaries or NCCL call: local ones are fused into the kernels' epilogues, "
                     f"remote ones {how} (CUDA IPC); tile-grid CTA plan inside each rank")
    else:
        plan = M.mm_one_piece_partition(N, N, N, world, quantum=nat.tile_shape(kid)[:3])
        ex = DistributedMM(plan, sr, CudaOps(sr, kid, st))
        C = torch.empty((N, N), dtype=torch.int32, device=dev)
        nred = sum(1 for t in plan.tasks if t.kind == "reduce" and rank in t.workers())

        def step():
            ex.run(A, B, C)
        launches_per_step = 2 + len(ex.temp_ids) + 3 * nred + len(ex.mine)
        plan_desc = (f"{world} GPUs, GPU-level mm_one_piece_partition(p={world}) "
                     f"({sum(1 for t in plan.tasks if t.kind == 'reduce')} k-cut NCCL MIN folds), "
                     "tile-grid CTA plan inside each rank")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # live roofline denominator: VIADDMNMX.U32 issue rate on this GPU
    tpc, probe_mhz = alu_peak(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        barrier()
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        barrier()
    ms_total = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms = ms_total / args.steps
    value = OPS_PER_STEP / (ms * 1e-3) / 1e9  # whole-job Gop/s

    # kernel-only timing of the dominant kernel on the same stream (1 GPU shape / this rank's cuboid)
    kern_ms = None
    if world == 1:
        kern_ms = ms  # the step is exactly one paco_mm launch
    clocks = clk.summary()

    # e2e: public API from pinned host buffers (H2D A, B, C; D2H C) -- rank 0's GPU, whole problem
    e2e = None
    if world == 1:
        C_h = torch.full((N, N), INF, dtype=torch.int32).pin_memory()
        M.mm_seq(A_h, B_h, C_h, sr)  # warm
        torch.cuda.synchronize(dev)
        t_e2e = []
        for _ in range(args.e2e_steps):
            C_h.fill_(INF)
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            f0.record(st)
            M.mm_seq(A_h, B_h, C_h, sr)
            f1.record(st)
            f1.synchronize()
            t_e2e.append(f0.elapsed_time(f1))
        e2e_ms = statistics.median(t_e2e)
        e2e = {"value": OPS_PER_STEP / (e2e_ms * 1e-3) / 1e9, "unit": "Gop/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": 3 * N * N * 4,
               "d2h_bytes_per_step": N * N * 4, "api": "paper_2011_01441_b200.matmul.mm_seq (pinned host numpy-equivalent tensors)"}
    elif args.fold == "fused":
        # every rank uploads the A/B blocks its cuboid reads (k-chunked, overlapped with
        # the folds into the owners' C) and reads its owned C rectangles back
        C_h = torch.empty((N, N), dtype=torch.int32).pin_memory()
        ex.run_host(A_h, B_h, C_h)  # warm
        t_e2e, nbytes = [], (0, 0)
        for _ in range(args.e2e_steps):
            barrier()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(st)
            nbytes = ex.run_host(A_h, B_h, C_h)
            f1.record(st)
            f1.synchronize()
            t = torch.tensor([f0.elapsed_time(f1)], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e.append(float(t.item()))
        tot = torch.tensor(list(nbytes), device=dev, dtype=torch.float64)
        dist.all_reduce(tot)
        e2e_ms = statistics.median(t_e2e)
        e2e = {"value": OPS_PER_STEP / (e2e_ms * 1e-3) / 1e9, "unit": "Gop/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(tot[0].item()), "d2h_bytes_per_step": int(tot[1].item()),
               "bytes": "summed over ranks; time = max over ranks",
               "api": "paper_2011_01441_b200.distributed.FusedDistributedMM.run_host (pinned host tensors)"}

    if rank == 0:
        peak_max = 2 * tpc * 148 * 1965.0 / 1e6  # Top/s at the 1965 MHz max SM clock
        traffic, traffic_src = ncu_traffic()
        achieved = OPS_PER_STEP / (kern_ms * 1e-3) / 1e12 if kern_ms else value / world / 1e3
        line = {
            "metric": METRIC, "value": value, "unit": "Gop/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded numpy default_rng(1002), BASELINE cfg2 distribution)",
            "config": {"workload": "cfg2: (min,+) saturating tropical MM n=m=k=8192, int32 [0,2^20) "
                                   "+ 10% INF=2^30 (BASELINE.json configs[1])",
                       "plan": plan_desc, "l2": "inputs 2 x 256 MiB > 126 MB L2 (no flush)",
                       "ops_per_step": OPS_PER_STEP},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_max, "unit": "Top/s",
                         "frac": achieved / peak_max,
                         "peak_source": (f"live VIADDMNMX.U32 probe: {tpc:.2f} terms/clk/SM x 2 op x 148 SM "
                                         f"x 1965 MHz max clock (probe ran at {probe_mhz:.0f} MHz)"),
                         "peak_at_run_clock": (2 * tpc * 148 * clocks["sm_mhz"] / 1e6) if clocks.get("sm_mhz") else None,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes": ALG_BYTES},
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

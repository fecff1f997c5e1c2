"""Command-line harness for the MM / Strassen path.

    python -m paper_2011_01441_b200.cli mm --n 2048 --m 2048 --k 2048 --p 3 --semiring minplus-sat --csv
    python -m paper_2011_01441_b200.cli strassen --n 4096 --p 7 --variant const-pieces --gamma 2 --csv
    python -m paper_2011_01441_b200.cli bench --spec sweep.txt --out runs.csv

One CSV row per run with the reference's stable header
``algo,n,m,k,p,Z,L,seed,mode,time_s,work_total,work_max,miss_total,miss_max,temp_peak,ok``
(+ ``plan_s``).  ``time_s`` is the min wall time of >= 3 repeats
around execute (device-synchronised); simulate mode (``serial_sim``) leaves it
empty as the spec's bench contract says.  ``Z``, ``L``, ``miss_*`` belong to the
cache simulator, which is out of scope on B200 (ncu counters replace it): empty.
``ok`` checks the result against ``mm_oracle`` -- the defining sums run as the
device naive kernel -- or, for Strassen, against classic (+,x) MM.  Exit code
is nonzero if any check fails.  Only the MM and Strassen algorithms exist here
(the reference's LCS / GAP / sort modules are outside this build's scope).
"""

from __future__ import annotations

import argparse
import sys
import time

import numpy as np
import torch

from . import matmul as M
from . import strassen as S
from .plan import PlanError

HEADER = ("algo,n,m,k,p,Z,L,seed,mode,time_s,work_total,work_max,miss_total,miss_max,"
          "temp_peak,ok,plan_s")

SEMIRINGS = {
    "int": M.SEMIRING_INT, "f64": M.SEMIRING_F64, "minplus": M.SEMIRING_MINPLUS,
    "minplus-sat": M.SEMIRING_MINPLUS_SAT, "maxplus": M.SEMIRING_MAXPLUS,
    "f32": M.SEMIRING_F32, "bf16": M.SEMIRING_BF16,
}
MODES = ("serial_sim", "parallel")


def _operands(semiring_name: str, n: int, m: int, k: int, seed: int):
    """Seeded inputs in each semiring's natural domain (BASELINE.json's draws)."""
    rng = np.random.default_rng(seed)
    if semiring_name == "int":
        return rng.integers(-8, 9, (n, k), dtype=np.int32), rng.integers(-8, 9, (k, m), dtype=np.int32)
    if semiring_name in ("minplus", "minplus-sat"):
        a = rng.integers(0, 2**20, (n, k), dtype=np.int32)
        a[rng.random(a.shape) < 0.1] = 2**30
        b = rng.integers(0, 2**20, (k, m), dtype=np.int32)
        b[rng.random(b.shape) < 0.1] = 2**30
        if semiring_name == "minplus":
            a, b = a.astype(np.int64), b.astype(np.int64)
        return a, b
    if semiring_name == "maxplus":
        return (rng.integers(-2**20, 2**20, (n, k), dtype=np.int32),
                rng.integers(-2**20, 2**20, (k, m), dtype=np.int32))
    if semiring_name == "bf16":
        a = torch.from_numpy(rng.standard_normal((n, k), dtype=np.float32)).to(torch.bfloat16)
        b = torch.from_numpy(rng.standard_normal((k, m), dtype=np.float32)).to(torch.bfloat16)
        return a.cuda(), b.cuda()
    dt = np.float64 if semiring_name == "f64" else np.float32
    return rng.uniform(-1, 1, (n, k)).astype(dt), rng.uniform(-1, 1, (k, m)).astype(dt)


def _close(semiring_name: str, got, want) -> bool:
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else got
    want = want.cpu().numpy() if isinstance(want, torch.Tensor) else want
    if semiring_name in ("f64", "f32", "bf16"):
        ref = want.astype(np.float64)
        den = max(np.linalg.norm(ref), 1e-300)
        return bool(np.linalg.norm(got.astype(np.float64) - ref) / den <= 1e-5)
    return bool(np.array_equal(got, want))


def _timed(fn, repeats: int) -> float:
    best = float("inf")
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def _row(algo, n, m, k, p, seed, mode, time_s, rep, ok, plan_s) -> str:
    t = "" if time_s is None else f"{time_s:.6f}"
    return ",".join(str(x) for x in (
        algo, n, m, k, p, "", "", seed, mode, t, rep.work_total, rep.work_max, "", "",
        rep.temp_space_peak, "pass" if ok else "fail", f"{plan_s:.6f}"))


def run_mm(n: int, m: int, k: int, p: int, *, variant: str = "paco", weights=None,
           semiring: str = "int", seed: int = 0, mode: str = "serial_sim", repeats: int = 3,
           devices=None, base: int = 32) -> tuple[str, bool]:
    if semiring not in SEMIRINGS:
        raise ValueError(f"unknown semiring {semiring!r} (one of {', '.join(SEMIRINGS)})")
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    sr = SEMIRINGS[semiring]
    t0 = time.perf_counter()
    if variant == "paco":
        plan = M.mm_paco_partition(n, m, k, p, base=base)
    elif variant == "one-piece":
        plan = M.mm_one_piece_partition(n, m, k, p)
    elif variant == "hetero":
        w = tuple(weights) if weights else (M.measured_weights(devices) if devices else (1.0,) * p)
        if len(w) != p:
            raise ValueError(f"--weights has {len(w)} entries, p={p}")
        plan = M.mm_hetero_partition(n, m, k, w)
    else:
        raise ValueError(f"unknown variant {variant!r}")
    plan_s = time.perf_counter() - t0
    A, B = _operands(semiring, n, m, k, seed)
    dev = torch.cuda.current_device()
    A_d = A if isinstance(A, torch.Tensor) else torch.from_numpy(A).cuda(dev)
    B_d = B if isinstance(B, torch.Tensor) else torch.from_numpy(B).cuda(dev)
    zero = sr.zero
    cdt = {"int": torch.int64, "f64": torch.float64, "minplus": torch.int64, "minplus-sat": torch.int32,
           "maxplus": torch.int32, "f32": torch.float32, "bf16": torch.float32}[semiring]
    C = torch.full((n, m), zero, dtype=cdt, device=dev)
    rep = M.mm_execute(plan, A_d, B_d, C, sr, mode=mode, devices=devices)
    want = M.mm_oracle(A_d, B_d, sr)
    ok = _close(semiring, C, want)

    def again():
        C.fill_(zero)
        M.mm_execute(plan, A_d, B_d, C, sr, mode=mode, devices=devices)

    time_s = None if mode == "serial_sim" else _timed(again, max(3, repeats))
    return _row("mm", n, m, k, p, seed, mode, time_s, rep, ok, plan_s), ok


def run_strassen(n: int, p: int, *, variant: str = "paco", gamma: int = 8, seed: int = 0,
                 mode: str = "serial_sim", repeats: int = 3, devices=None, base: int | None = None,
                 split_leftover: bool = False) -> tuple[str, bool]:
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    t0 = time.perf_counter()
    # GPU default: two Strassen levels (leaves of n/4, as cfg5) -- the API's
    # reference default of 64 would launch 7^log2(n/64) tiny leaf products
    b = base if base is not None else max(S.DEFAULT_STRASSEN_BASE, n // 4)
    if variant == "paco":
        plan = S.strassen_paco_partition(n, p, base=b, split_leftover=split_leftover)
    elif variant == "const-pieces":
        plan = S.strassen_const_pieces_partition(n, p, S.SuperRoundCfg(gamma=gamma), base=b)
    else:
        raise ValueError(f"unknown variant {variant!r}")
    plan_s = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    dev = torch.cuda.current_device()
    A = torch.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32)).cuda(dev)
    B = torch.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32)).cuda(dev)
    C, rep = S.strassen_execute(plan, A, B, mode=mode, devices=devices, with_report=True)
    want = M.mm_oracle(A.double(), B.double(), M.SEMIRING_F64)
    got = C.double().cpu().numpy()
    ref = want.cpu().numpy() if isinstance(want, torch.Tensor) else want
    ok = bool(np.linalg.norm(got - ref) <= 1e-4 * np.linalg.norm(ref))
    time_s = None if mode == "serial_sim" else _timed(
        lambda: S.strassen_execute(plan, A, B, mode=mode, devices=devices), max(3, repeats))
    return _row("strassen", n, n, n, p, seed, mode, time_s, rep, ok, plan_s), ok


def _ints(text: str) -> list[int]:
    return [int(x) for x in str(text).split(",") if x.strip()]


def run_spec(spec: dict, out) -> bool:
    """`paco bench`: sweep lists of n and p; one row each."""
    algo = spec.get("algo", "mm")
    if algo not in ("mm", "strassen"):
        raise ValueError(f"algo {algo!r} is outside this build (mm, strassen)")
    repeats = int(spec.get("repeats", 3))
    mode = spec.get("mode", "parallel")
    if mode != "serial_sim" and repeats < 3:
        raise ValueError("timing mode needs repeats >= 3 (min of at least three runs)")
    seed = int(spec.get("seed", 0))
    all_ok = True
    print(HEADER, file=out)
    for n in _ints(spec.get("n", "256")):
        for p in _ints(spec.get("p", "1")):
            if algo == "mm":
                row, ok = run_mm(n, int(spec.get("m", n)), int(spec.get("k", n)), p,
                                 variant=spec.get("variant", "paco"), semiring=spec.get("semiring", "int"),
                                 seed=seed, mode=mode, repeats=repeats)
            else:
                row, ok = run_strassen(n, p, variant=spec.get("variant", "paco"),
                                       gamma=int(spec.get("gamma", 8)), seed=seed, mode=mode, repeats=repeats,
                                       base=int(spec["base"]) if "base" in spec else None,
                                       split_leftover=spec.get("split_leftover", "0") in ("1", "true", "yes"))
            print(row, file=out, flush=True)
            all_ok &= ok
    return all_ok


def read_spec(path: str) -> dict:
    spec = {}
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                key, _, val = line.partition("=")
                spec[key.strip()] = val.strip()
    return spec


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paco")
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("mm")
    a.add_argument("--n", type=int, required=True)
    a.add_argument("--m", type=int)
    a.add_argument("--k", type=int)
    a.add_argument("--p", type=int, required=True)
    a.add_argument("--variant", default="paco", choices=["paco", "one-piece", "hetero"])
    a.add_argument("--weights", help="comma-separated worker throughputs (hetero)")
    a.add_argument("--semiring", default="int", choices=sorted(SEMIRINGS))
    s = sub.add_parser("strassen")
    s.add_argument("--n", type=int, required=True)
    s.add_argument("--p", type=int, required=True)
    s.add_argument("--gamma", type=int, default=8)
    s.add_argument("--variant", default="paco", choices=["paco", "const-pieces"])
    s.add_argument("--base", type=int, help="leaf size (default max(64, n/4): two levels, as cfg5)")
    s.add_argument("--split-leftover", action="store_true",
                   help="cut the last < p leaves into p MM-1-Piece cuboids (paco variant)")
    for x in (a, s):
        x.add_argument("--seed", type=int, default=0)
        x.add_argument("--mode", default="serial_sim", choices=MODES)
        x.add_argument("--repeats", type=int, default=3)
        x.add_argument("--devices", help="comma-separated CUDA devices for the plan's workers")
        x.add_argument("--csv", action="store_true", help="print the CSV header and row")
    b = sub.add_parser("bench")
    b.add_argument("--spec", required=True)
    b.add_argument("--out", default="-")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "bench":
            out = sys.stdout if args.out == "-" else open(args.out, "w")
            try:
                ok = run_spec(read_spec(args.spec), out)
            finally:
                if out is not sys.stdout:
                    out.close()
            return 0 if ok else 1
        devices = _ints(args.devices) if args.devices else None
        if args.cmd == "mm":
            weights = [float(x) for x in args.weights.split(",")] if args.weights else None
            row, ok = run_mm(args.n, args.m or args.n, args.k or args.n, args.p, variant=args.variant,
                             weights=weights, semiring=args.semiring, seed=args.seed, mode=args.mode,
                             repeats=args.repeats, devices=devices)
        else:
            row, ok = run_strassen(args.n, args.p, variant=args.variant, gamma=args.gamma, seed=args.seed,
                                   mode=args.mode, repeats=args.repeats, devices=devices, base=args.base,
                                   split_leftover=args.split_leftover)
    except (PlanError, ValueError) as e:
        print(f"paco: error: {e}", file=sys.stderr)
        return 2
    if args.csv:
        print(HEADER)
        print(row)
    else:
        fields = dict(zip(HEADER.split(","), row.split(",")))
        print(" ".join(f"{k}={v}" for k, v in fields.items() if v != ""))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())

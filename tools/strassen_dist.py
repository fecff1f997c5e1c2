"""cfg5 (Strassen fp32, n=16384, 2 levels) over N GPUs, one process per GPU.

    python tools/strassen_dist.py                      # N=1
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29511 tools/strassen_dist.py [--size 16384] [--no-split]

Each rank forms its plan nodes' S/T from replicated A, B, multiplies them and
adds the signed products into a partial C; C is one NCCL reduce-scatter
(``distributed.DistributedStrassen``).  Timed region: ``run`` (forming,
products, partial sums, reduce-scatter), CUDA events, max over ranks.
Checks the gathered C against an fp64 product on a sample of rows.
"""

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

from paper_2011_01441_b200 import strassen as S
from paper_2011_01441_b200.distributed import CudaStrassenOps, DistributedStrassen


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--base", type=int, default=None, help="default n/4 (2 levels)")
    ap.add_argument("--no-split", action="store_true")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = torch.cuda.device_count()
    dev = local % ngpu
    torch.cuda.set_device(dev)
    if world > 1 or "MASTER_ADDR" in os.environ:
        dist.init_process_group("nccl" if world <= ngpu else "gloo", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev) if world <= ngpu else None)
    else:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", dev))
    n = args.size
    base = args.base or max(64, n // 4)
    plan = S.strassen_paco_partition(n, world, base=base, split_leftover=not args.no_split)
    g = torch.Generator(device="cuda").manual_seed(1005)
    a = torch.rand((n, n), device="cuda", generator=g) * 2 - 1
    b = torch.rand((n, n), device="cuda", generator=g) * 2 - 1
    ds = DistributedStrassen(plan, CudaStrassenOps(torch.float32))
    for _ in range(args.warmup):
        slab = ds.run(a, b)
    times = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        slab = ds.run(a, b)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t))
    C = ds.gather(slab)
    if rank == 0:
        rows = torch.arange(0, n, max(1, n // 64), device="cuda")
        ref = a[rows].double() @ b.double()
        err = float(torch.linalg.norm(C[rows].double() - ref) / torch.linalg.norm(ref))
        ms = statistics.median(times)
        alg = 49 * 2 * (n // 4) ** 3 + 18 * (n // 2) ** 2 + 7 * 18 * (n // 4) ** 2
        print(json.dumps({"workload": f"cfg5 Strassen fp32 n={n} base={base}", "n_gpus": world,
                          "variant": plan.meta["variant"], "ms": ms, "times": times,
                          "tflop_s_algorithmic": alg / ms / 1e9, "tflop_s_classic": 2 * n ** 3 / ms / 1e9,
                          "rel_err_sample_rows": err, "nodes_rank0": len(ds.nodes), "pieces_rank0": len(ds.pieces)}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

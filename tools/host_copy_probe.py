"""Host-side staging costs on the GPU box: pageable->pinned copy bandwidth vs
thread count, cudaHostRegister / Unregister of NumPy buffers, pinned H2D/D2H."""
import ctypes
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
res = {"cores": len(os.sched_getaffinity(0))}
N = 8192
src = np.random.default_rng(0).integers(0, 2**20, (N, N), dtype=np.int32)
dst_p = torch.empty((N, N), dtype=torch.int32, pin_memory=True).numpy()
dst_np = np.empty((N, N), np.int32)
dst_np.fill(1)
for T in (1, 2, 4, 8, 16, 24, 32):
    pool = ThreadPoolExecutor(T)
    cuts = [N * i // T for i in range(T + 1)]
    for name, dst in (("to_pinned", dst_p), ("to_pageable", dst_np)):
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            list(pool.map(lambda ab: np.copyto(dst[ab[0]:ab[1]], src[ab[0]:ab[1]]), zip(cuts[:-1], cuts[1:])))
            best = min(best, time.perf_counter() - t0)
        res[f"copy_{name}_T{T}_GBs"] = src.nbytes / best / 1e9
    # strided column chunk (A[:, l0:l1] with 2048 columns)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        list(pool.map(lambda ab: np.copyto(dst_p[ab[0]:ab[1], :2048], src[ab[0]:ab[1], :2048]), zip(cuts[:-1], cuts[1:])))
        best = min(best, time.perf_counter() - t0)
    res[f"copy_cols2048_T{T}_GBs"] = src.nbytes / 4 / best / 1e9
    pool.shutdown()
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
torch.cuda.init()
lib = ctypes.CDLL(None)
try:
    cudart = ctypes.CDLL("libcudart.so")
except OSError:
    import glob
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*"))
    cudart = ctypes.CDLL(cands[0]) if cands else None
if cudart is not None:
    for trial in range(3):
        a = np.empty((N, N), np.int32)
        a.fill(3)
        t0 = time.perf_counter()
        rc = cudart.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 0)
        t1 = time.perf_counter()
        rc2 = cudart.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
        t2 = time.perf_counter()
        res[f"register_256MiB_ms_{trial}"] = (t1 - t0) * 1e3
        res[f"unregister_256MiB_ms_{trial}"] = (t2 - t1) * 1e3
        res["register_rc"] = (rc, rc2)
d = torch.empty((N, N), dtype=torch.int32, device="cuda")
hp = torch.from_numpy(dst_p)
for name, fn in (("h2d_pinned", lambda: d.copy_(hp, non_blocking=True)), ("d2h_pinned", lambda: hp.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    res[f"{name}_GBs"] = 5 * src.nbytes / (time.perf_counter() - t0) / 1e9
print(json.dumps(res, indent=1))

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2011_01441_b200 import matmul as M
rng = np.random.default_rng(0)
n, m, k = 200, 150, 300
A = rng.uniform(-1, 1, (n, k)).astype(np.float32); B = rng.uniform(-1, 1, (k, m)).astype(np.float32)
ref = A.astype(np.float64) @ B.astype(np.float64)
for sr in (M.SEMIRING_F32, M.SEMIRING_F32_SIMT):
    for name, plan in (("paco", M.mm_paco_partition(n, m, k, 3)), ("one", M.mm_one_piece_partition(n, m, k, 3)), ("one1", M.mm_one_piece_partition(n, m, k, 1))):
        for mode in ("serial_sim", "parallel"):
            C = torch.zeros((n, m), device="cuda")
            M.mm_execute(plan, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C, sr, mode=mode)
            got = C.cpu().numpy().astype(np.float64)
            print(sr.name, name, mode, np.linalg.norm(got - ref) / np.linalg.norm(ref), np.abs(got-ref).max())
    o = M.mm_oracle(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), sr).cpu().numpy()
    print("oracle", np.linalg.norm(o - ref) / np.linalg.norm(ref))

import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2011_01441_b200 import matmul as M
n=m=128; k=32
A = np.tile(np.arange(k,dtype=np.float32),(n,1)); B = np.ones((k,m),np.float32)
C = np.full((n, m), 7, np.float32)
M.mm_seq(A, B, C, M.SEMIRING_F32, overwrite=True)
print("tf32 overwrite sentinel C[0,:4]", C[0,:4], "want 496", flush=True)
C = np.full((n, m), 7, np.float32)
M.mm_seq(A, B, C, M.SEMIRING_F32)
print("tf32 accumulate sentinel C[0,:4]", C[0,:4], "want 503", flush=True)
a = torch.from_numpy(A).cuda().to(torch.bfloat16); b = torch.from_numpy(B).cuda().to(torch.bfloat16)
c = torch.full((n, m), 7., device="cuda")
M.mm_seq(a, b, c, M.SEMIRING_BF16)
print("bf16 C[0,:4]", c[0,:4].cpu().numpy(), "want 503", flush=True)

"""One cfg5 Strassen call inside a cudaProfilerStart/Stop range (for an ncu
launch list: ncu --profile-from-start off --metrics gpu__time_duration.sum)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import strassen as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a = torch.rand(n, n, device="cuda") * 2 - 1
b = torch.rand(n, n, device="cuda") * 2 - 1
S.strassen_seq(a, b, n, base=n // 4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
S.strassen_seq(a, b, n, base=n // 4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")

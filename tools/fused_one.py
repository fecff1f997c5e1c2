"""One cfg5 leaf-level launch of the fused-formation 3xTF32 kernel (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import strassen as S
from paper_2011_01441_b200.device import View

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192   # a level-1 node: 7 leaf products of n/2
mode = sys.argv[2] if len(sys.argv) > 2 else "fused"   # fused | split | raw | b3 | b3n
S.FUSED_PRODUCER = mode == "fused"
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
c = torch.zeros(n, n, device="cuda")
st = torch.cuda.current_stream()
for _ in range(2):
    if mode == "b3n":   # bf16x3, B in its own layout (the cfg5 default)
        S._leaf_level_b3(View.of(a), View.of(b), [(View.of(c), 1)], st, bnat=True)
    elif mode == "b3":
        S._leaf_level_b3(View.of(a), View.of(b.t().contiguous()), [(View.of(c), 1)], st)
    elif mode == "raw":
        S._leaf_level_b2raw(View.of(a),
                            View.of(b.t().contiguous()), [(View.of(c), 1)], st)
    elif S.FUSED_PRODUCER:
        S._leaf_level_fused(View.of(a), View.of(b.t().contiguous()), [(View.of(c), 1)], st)
    else:
        S._leaf_level_multi(View.of(a), View.of(b), [(View.of(c), 1)], st)
torch.cuda.synchronize()
print("ok")

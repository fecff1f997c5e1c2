"""The library's launches captured into CUDA graphs (torch.cuda.graph), with the
capture as the process's FIRST library call: no pool / allocation / attribute
call may break the capture, and replays must match eager launches bit for bit.
Runs in a fresh subprocess so the library's one-time set-up happens inside the
capture."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import torch
sys.path.insert(0, sys.argv[1])
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

g0 = torch.Generator(device="cuda").manual_seed(3)
a = torch.randn(1000, 256, device="cuda", generator=g0).to(torch.bfloat16)
b = torch.randn(256, 520, device="cuda", generator=g0).to(torch.bfloat16)
# min-plus on a view whose row pitch is not 16-byte aligned (the repack path)
ai = torch.randint(0, 1 << 20, (300, 301), device="cuda", dtype=torch.int32, generator=g0)
bi = torch.randint(0, 1 << 20, (301, 130), device="cuda", dtype=torch.int32, generator=g0)
av, bv = View.of(ai[:, :299]), View.of(bi[:299])
c_cap = torch.empty(1000, 520, device="cuda")
ci_cap = torch.full((300, 130), 2**30, device="cuda", dtype=torch.int32)
torch.cuda.synchronize()
cap = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=cap):
    launch_mm(nat.SR_BF16_F32, cap, View.of(a), View.of(b), View.of(c_cap), overwrite=True)
    launch_mm(nat.SR_MINPLUS_SAT32, cap, av, bv, View.of(ci_cap), overwrite=True)
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
c = torch.empty_like(c_cap)
ci = torch.full_like(ci_cap, 2**30)
st = torch.cuda.current_stream()
launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
launch_mm(nat.SR_MINPLUS_SAT32, st, av, bv, View.of(ci), overwrite=True)
torch.cuda.synchronize()
ref = a.double() @ b.double()
assert float((c.double() - ref).norm() / ref.norm()) < 1e-5
assert torch.equal(c, c_cap), "bf16 replay differs from the eager launch"
assert torch.equal(ci, ci_cap), "min-plus replay differs from the eager launch"
print("ok")
"""


def test_graph_capture_first_call():
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]

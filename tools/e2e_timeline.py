"""Timeline of the pinned-host pipeline: when each copy / kernel starts and ends."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import mm as MM

n = 8192
A = torch.randint(0, 2**20, (n, n), dtype=torch.int32).pin_memory()
B = torch.randint(0, 2**20, (n, n), dtype=torch.int32).pin_memory()
C = torch.full((n, n), 2**30, dtype=torch.int32).pin_memory()
for _ in range(2):
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
# instrument: monkeypatch launch_mm and _copy2d to record events
rec = []
orig_launch, orig_copy, orig_fold = MM.launch_mm, MM._copy2d, MM.launch_fold
def ev(stream):
    e = torch.cuda.Event(enable_timing=True); e.record(stream); return e
def launch(kid, st, a, b, c, **kw):
    e0 = ev(st); orig_launch(kid, st, a, b, c, **kw); rec.append(("kernel %dx%dx%d" % (c.rows, c.cols, a.cols), e0, ev(st)))
def copy(st, dst, *args):
    e0 = ev(st); orig_copy(st, dst, *args); rec.append(("%s %dx%d" % ("H2D" if dst.is_cuda else "D2H", args[-2], args[-1]), e0, ev(st)))
def fold(kid, st, dst, src, reset):
    e0 = ev(st); orig_fold(kid, st, dst, src, reset); rec.append(("fold", e0, ev(st)))
MM.launch_mm, MM._copy2d, MM.launch_fold = launch, copy, fold
start = ev(torch.cuda.current_stream())
M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
end = ev(torch.cuda.current_stream()); end.synchronize()
print("total %.2f ms" % start.elapsed_time(end))
for name, e0, e1 in rec:
    print("%-22s start %7.2f  end %7.2f  dur %6.2f" % (name, start.elapsed_time(e0), start.elapsed_time(e1), e0.elapsed_time(e1)))

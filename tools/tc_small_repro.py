"""Single 3xTF32 launches on small odd shapes / offset views (dev tool)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2011_01441_b200 import _native as nat
if os.environ.get("PACO_LIB"):  # an older build: bind only the symbols it has
    import ctypes
    _probe = ctypes.CDLL(nat.LIB_PATH)
    nat.SIGNATURES = {k: v for k, v in nat.SIGNATURES.items() if hasattr(_probe, k)}
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm
torch.manual_seed(0)
SR = nat.SR_BF16_F32 if os.environ.get("BF16") else nat.SR_F32_TC
big_a = torch.randn(256, 256, device="cuda"); big_b = torch.randn(256, 256, device="cuda")
if os.environ.get("BF16"):
    big_a, big_b = big_a.to(torch.bfloat16), big_b.to(torch.bfloat16)
cases = [tuple(int(x) for x in c.split(",")) for c in sys.argv[1:]] or [
    (0, 0, 25, 64, 0, 32), (25, 0, 39, 64, 0, 21), (25, 0, 39, 32, 21, 43), (25, 32, 39, 32, 21, 43)]
for (i0, l0, n, k, j0, m) in cases:
    for tgt in ("fresh", "view"):
        big_c = torch.zeros(256, 256, device="cuda")
        c = View.of(big_c).sub(i0, j0, n, m) if tgt == "view" else View.of(torch.zeros(n, m, device="cuda"))
        a = View.of(big_a).sub(i0, l0, n, k); b = View.of(big_b).sub(l0, j0, k, m)
        try:
            launch_mm(SR, torch.cuda.current_stream(), a, b, c, overwrite=True)
            torch.cuda.synchronize()
            ref = (big_a.float()[i0:i0 + n, l0:l0 + k] @ big_b.float()[l0:l0 + k, j0:j0 + m])
            got = big_c[i0:i0 + n, j0:j0 + m] if tgt == "view" else c.tensor[:n, :m]
            print("ok", (i0, l0, n, k, j0, m), tgt, "err %.1e" % float((got - ref).abs().max()), flush=True)
        except Exception as e:
            print("FAIL", (i0, l0, n, k, j0, m), tgt, str(e)[-60:], flush=True)
            sys.exit(1)

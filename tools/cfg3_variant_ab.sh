# cfg3 tcgen05 variants: default (1 CTA/SM, N = 256) vs PACO_TC_RES2=1 (2 CTAs/SM, N = 128)
python - <<'PY'
import os, subprocess, json
for r in (0, 1, 0, 1):
    env = dict(os.environ, PACO_DEV_KNOBS="1", PACO_TC_RES2=str(r))
    out = subprocess.run(["python", "tools/tc_graph_vs_eager.py"], env=env, capture_output=True, text=True)
    print("res2", r, out.stdout.strip(), out.stderr.strip()[-300:])
PY
PACO_DEV_KNOBS=1 PACO_TC_RES2=1 python - <<'PY'
import torch, sys
sys.path.insert(0, ".")
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm
g = torch.Generator(device="cuda").manual_seed(0)
for n, m, k in ((65536, 1024, 256), (1000, 520, 200), (4096, 384, 64)):
    a = torch.randn(n, k, device="cuda", generator=g).bfloat16()
    b = torch.randn(k, m, device="cuda", generator=g).bfloat16()
    c = torch.empty(n, m, device="cuda")
    launch_mm(nat.SR_BF16_F32, torch.cuda.current_stream(), View.of(a), View.of(b), View.of(c), overwrite=True)
    ref = a.double() @ b.double()
    print(n, m, k, "rel err", float((c.double() - ref).norm() / ref.norm()))
PY

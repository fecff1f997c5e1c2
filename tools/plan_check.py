import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
"""CTA plan shape statistics (balance, tile visits, k-cut pieces) per k weight (PACO_CTA_KW)."""
from paper_2011_01441_b200 import _native as nat
from collections import Counter
import sys
for (n,m,k) in [(8192,8192,8192),(8192,8192,256),(1024,8192,2048),(16384,16384,16384),(3000,5000,7000),(65536,1024,256),(2048,4096,8192)]:
    out=[]
    for p in [1184, 2048, 4096]:
        try:
            pcs = nat.plan_cta(nat.SR_MINPLUS_SAT32, n,m,k,p)
        except Exception as e:
            out.append(f"p={p}: infeasible"); continue
        vols = [q[3]*q[4]*q[5] for q in pcs]
        mean = sum(vols)/len(vols)
        visits = sum(q[3]*q[4] for q in pcs)
        out.append(f"p={p}: max/mean {max(vols)/mean:.3f} visits {visits} kcut {sum(q[5]!=-(-k//16) for q in pcs)}")
    print((n,m,k), " | ".join(out))

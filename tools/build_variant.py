"""Build a variant of libpaco_b200.so with extra -D defines into variants/<name>.so
(git-ignored, travels to the GPU box), for A/B runs with PACO_LIB=variants/<name>.so.
Usage: python tools/build_variant.py <name> -DPACO_PAIR_CG=1 [...]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "variants")
obj_dir = os.path.join(out_dir, name + "_obj")
os.makedirs(obj_dir, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(G.PKG, "csrc", "*.cu")))
objs = [os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o") for s in srcs]
procs = [subprocess.Popen([G._nvcc()] + G.NVCC_FLAGS + defs + ["-c", s, "-o", o]) for s, o in zip(srcs, objs)]
if any(p.wait() != 0 for p in procs):
    sys.exit("nvcc failed")
lib = os.path.join(out_dir, name + ".so")
subprocess.run([G._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + objs, check=True)
print(lib)

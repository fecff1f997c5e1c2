"""All paco_alu_probe kinds: issue rate per SM and the implied peak (dev tool)."""
import sys, os, ctypes
sys.path.insert(0, os.getcwd())
from paper_2011_01441_b200 import _native as nat
lib = nat.load()
for which, name in ((0, "viaddmnmx.u32"), (1, "viaddmnmx.s32"), (2, "ffma"), (3, "dfma")):
    tpc = ctypes.c_double(); mhz = ctypes.c_double()
    nat.check(lib.paco_alu_probe(0, None, which, 20000, ctypes.byref(tpc), ctypes.byref(mhz)))
    print(f"{name}: {tpc.value:.2f} terms/clk/SM at {mhz.value:.0f} MHz -> {2*tpc.value*148*mhz.value/1e6:.1f} T(fl)op/s")

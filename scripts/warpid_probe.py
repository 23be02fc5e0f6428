"""Experiment: hardware warp slots (%warpid) of two co-resident 8-warp CTAs."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
from paper_2507_22195_b200 import _native
lib = _native.load()
nb = 296
buf = (C.c_int * (nb * 16))()
lib.mhdg_debug_warpid(buf, C.c_int(nb))
by_sm = {}
for b in range(nb):
    for w in range(8):
        sm, wid = buf[(b * 8 + w) * 2], buf[(b * 8 + w) * 2 + 1]
        by_sm.setdefault(sm, []).append((b, w, wid))
for sm in sorted(by_sm)[:4]:
    print(sm, by_sm[sm])

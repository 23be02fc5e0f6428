import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
from paper_2507_22195_b200 import _native
lib = _native.load()
lib.mhdg_debug_gj8.restype = C.c_double
print({v: round(lib.mhdg_debug_gj8(C.c_int(v)), 1) for v in (0, 1, 2)})

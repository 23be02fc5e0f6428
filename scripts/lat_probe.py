"""Experiment: dependent-chain latencies on the B200 (timing build)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
from paper_2507_22195_b200 import _native
lib = _native.load()
lib.mhdg_debug_latency.restype = C.c_double
names = {-1: "dfma", 0: "log+add", 1: "exp*mul", 2: "ddiv", 3: "dmma_dependent", 4: "dmma_4chains_per_dmma",
         10: "shfl64+add", 11: "drcp+add", 12: "redux+cvt+add", 13: "bar.sync128+add"}
print(json.dumps({v: round(lib.mhdg_debug_latency(C.c_int(k)), 1) for k, v in names.items()}))
lib.mhdg_debug_contend.restype = C.c_double
res = {}
for mode, mn in ((0, "dfma"), (1, "shfl+add"), (2, "int3")):
    for other, on in ((9, "alone"), (4, "same_sched"), (1, "other_sched")):
        for dm, dn in ((1, "dmma"), (0, "dfma")):
            if other == 9 and dm == 0:
                continue
            ops = C.c_double(0)
            lat = lib.mhdg_debug_contend(C.c_int(mode), C.c_int(other), C.c_int(dm), C.byref(ops))
            res[f"{mn}|{on}|{dn if other != 9 else '-'}"] = [round(lat, 1), round(ops.value, 4)]
print(json.dumps(res, indent=1))

import sys, os, math
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import __graft_entry__; __graft_entry__.build()
import numpy as np, torch
from test_gpu_krylov_engine import _disc, _system, _rel
from paper_2507_22195_b200 import solver
mode = sys.argv[1]
kw = dict(rel_tol=float(sys.argv[2]), restart=int(sys.argv[3]))
case, disc = _disc()
lin, res = _system(disc, case, dt=0.25)
try:
    if mode == 'host':
        x, s = solver.solve_condensed_host(lin, res, **kw)
    else:
        x, s = solver.solve_condensed(lin, res, **kw)
    torch.cuda.synchronize()
    print(mode, kw, s.outer_iterations, s.inner_iterations, s.converged, s.rel_residual, flush=True)
except Exception as e:
    print(mode, kw, 'EXC', repr(e), flush=True)

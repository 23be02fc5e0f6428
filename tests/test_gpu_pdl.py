"""Programmatic dependent launch is an overlap optimisation only: the
library built with -DMHDG_PDL=0 (no griddepcontrol.wait, no launch
attribute) must produce bit-identical condensed matvec, condensed rhs,
recovery and preconditioner outputs, inviscid and viscous (the
pdl_wait invariant documented in mhdg_kernels.cuh is otherwise unchecked).
Builds the variant library (about a minute of nvcc) into a temporary
directory and runs both in subprocesses."""

import json
import os
import subprocess
import sys
import tempfile

import pytest

from helpers import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SCRIPT = r'''
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel, TaylorGreen
from paper_2507_22195_b200.assembly import StageContext
from paper_2507_22195_b200.mesh import build_box_macro_mesh
out = {}
gas = GasModel(1.4)
tg = TaylorGreen(mach=0.1, gas=gas)
for visc in (None, tg.viscous_params(1600.0, prandtl=0.71)):
    disc = Discretization(build_box_macro_mesh(tg.box, 3, 1), p=3, gas=gas,
                          flux=DissipationSpec("kepes"), viscosity=visc, device="cuda:0")
    f = disc.project(tg.initial)
    rng = np.random.default_rng(5)
    f.trace = f.trace * torch.from_numpy(1 + 0.01 * rng.standard_normal(tuple(f.trace.shape))).cuda()
    if visc is not None:
        f.q = disc.solve_gradient(f)
    alpha = 0.4358665215 / 0.57
    st = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(f), dt=0.57)
    res = disc.residuals(f, st)
    lin = disc.jacobian(f, st, ptc_weight=1.0)
    x = torch.from_numpy(rng.standard_normal(lin.trace_shape)).cuda()
    vals = dict(matvec=lin.matvec(x), rhs=lin.condensed_rhs(res), rec=lin.recover(res, x)[0],
                pre=lin.apply_preconditioner(x))
    key = "visc" if visc is not None else "inv"
    out[key] = {k: hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for k, v in vals.items()}
print(json.dumps(out))
'''


def _run(lib):
    env = dict(os.environ, MHDG_LIB=lib)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.timeout(1800)
def test_pdl_off_is_bit_identical(cuda_ok):
    import __graft_entry__

    with tempfile.TemporaryDirectory() as d:
        lib = os.path.join(d, "libmhdg_b200_nopdl.so")
        cmd = [__graft_entry__._nvcc()] + __graft_entry__.NVCC_FLAGS + ["-DMHDG_PDL=0", "-o", lib,
                                                                        os.path.join(__graft_entry__.CSRC,
                                                                                     "mhdg_capi.cu")]
        subprocess.run(cmd, check=True, timeout=900)
        off = _run(lib)
    on = _run(__graft_entry__.LIB)
    assert on == off

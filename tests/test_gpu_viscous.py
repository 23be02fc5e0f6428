"""GPU parity of the viscous operator (gradient unknowns q, level-1
condensation) against the reference's viscous goldens
(tests/golden/visc_*.npz): residual (r_w, r_trace, r_q), solve_gradient,
condensed matvec / rhs / recovery (d_w, d_q), face-block preconditioner.
Tolerances as in test_gpu_parity.py (max(floor, 10 x reference 1-ulp
sensitivity))."""

import numpy as np
import pytest

from helpers import golden_mesh, load_golden, rel

pytestmark = pytest.mark.gpu

CASES = ["visc_k1_kepes_entr", "visc_k2_kepes_entr", "visc_k3_es_entr", "visc_k2_lf_cons",
         "visc_tgv_k3_kepes"]


def tol(z, key, floor):
    return max(floor, 10.0 * float(z.get(f"sens_{key}", 0.0)))


@pytest.fixture(scope="module", params=CASES)
def case(request, cuda_ok):
    from paper_2507_22195_b200 import (Discretization, DissipationSpec, GasModel, StageContext,
                                       ViscousParams)
    from paper_2507_22195_b200.assembly import FieldSet

    z = load_golden(request.param)
    vp = ViscousParams(float(z["reynolds"]), float(z["mach"]), float(z["prandtl"]), float(z["mu"]))
    disc = Discretization(golden_mesh(z), p=int(z["p"]), gas=GasModel(1.4),
                          formulation=str(z["formulation"]), flux=DissipationSpec(str(z["flux"])),
                          viscosity=vp, device="cuda:0")
    fields = FieldSet(z["w"], z["trace"], z["q"])
    stage = StageContext(alpha=float(z["alpha"]), offset=z["offset"])
    res = disc.residuals(fields, stage)
    lin = disc.jacobian(fields, stage, ptc_weight=float(z["ptc"]))
    return request.param, z, disc, fields, res, lin


def test_viscous_residual(case):
    name, z, disc, fields, res, lin = case
    assert rel(res.r_w, z["r_w"]) <= tol(z, "r_w", 1e-12), name
    assert rel(res.r_trace, z["r_trace"]) <= tol(z, "r_trace", 1e-12), name
    assert rel(res.r_q, z["r_q"]) <= tol(z, "r_q", 1e-12), name


def test_solve_gradient(case):
    name, z, disc, fields, res, lin = case
    assert rel(disc.solve_gradient(fields), z["qgrad"]) <= tol(z, "qgrad", 1e-12), name


def test_viscous_condensed_operator(case):
    name, z, disc, fields, res, lin = case
    assert rel(lin.matvec(z["x"]), z["matvec"]) <= tol(z, "matvec", 1e-11), name
    assert rel(lin.condensed_rhs(res), z["rhs"]) <= tol(z, "rhs", 1e-11), name
    d_w, d_q = lin.recover(res, z["x"])
    assert rel(d_w, z["recover"]) <= tol(z, "recover", 1e-11), name
    assert rel(d_q, z["recover_q"]) <= tol(z, "recover_q", 1e-11), name
    assert rel(lin.apply_preconditioner(z["x"]), z["precond"]) <= tol(z, "precond", 1e-11), name

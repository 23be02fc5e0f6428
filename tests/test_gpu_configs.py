"""Parity on the BASELINE configs 2 and 3 against goldens produced by the
reference itself (tests/golden/make_golden.py --only-cfg3 / --only-cfg2-step):

  cfg3_ops_n4    inviscid Taylor-Green M=0.1, KEPES, k=3, n=4 (384 macros):
                 projected initial condition (bit-exact, CPU test) and the
                 residual / condensed operators at stage 1 of dt=0.57
  cfg3_step_n2   the first accepted DIRK(3,3) step at n=2 with dt=2.28 and
                 NewtonParams(max_iters=16): the reference rejects the step
                 twice (stage 1 needs 17 Newton iterations) and accepts
                 dt=0.57; the device must take the same path
  cfg2_step_n8   isentropic vortex, ES, k=3, n=8 (3,072 macros), one DIRK step

Tolerances: residual <= max(1e-12, 10x the reference's own
1-ulp sensitivity), condensed operators <= max(1e-11, 10x sensitivity),
converged states 1e-10, integrals 1e-12 relative, identical Newton counts
and the sign of the entropy change."""

import numpy as np
import pytest

from helpers import load_golden, rel

KEYS = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")


def _tgv(n):
    from paper_2507_22195_b200 import GasModel, TaylorGreen
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    tg = TaylorGreen(mach=0.1, gas=gas)
    return gas, tg, build_box_macro_mesh(tg.box, n, 1)


def test_cfg3_projection_bit_exact():
    """Host tables + gas algebra reproduce the reference's projected state."""
    from paper_2507_22195_b200.tables import HDGTables

    z = load_golden("cfg3_ops_n4")
    gas, tg, mesh = _tgv(4)
    t = HDGTables(mesh, 3)
    w = gas.entropy_vars(tg.initial(t.node_coords))
    tr = gas.entropy_vars(tg.initial(t.trace_coords))
    assert np.array_equal(w, z["w"]) and np.array_equal(tr, z["trace"])


@pytest.mark.gpu
def test_cfg3_operator_n4(cuda_ok):
    from paper_2507_22195_b200 import Discretization, DissipationSpec
    from paper_2507_22195_b200.assembly import StageContext

    z = load_golden("cfg3_ops_n4")
    gas, tg, mesh = _tgv(4)
    disc = Discretization(mesh, p=3, gas=gas, formulation="entropy",
                          flux=DissipationSpec("kepes"), device="cuda:0")
    fields = disc.project(tg.initial)
    assert rel(fields.w, z["w"]) == 0.0 and rel(fields.trace, z["trace"]) == 0.0
    vqs = disc.volume_quad_states(fields)
    assert rel(vqs, z["vqs"]) <= 1e-14
    alpha = float(z["alpha"])
    stage = StageContext(alpha=alpha, offset=z["offset"])
    res = disc.residuals(fields, stage)
    lin = disc.jacobian(fields, stage, ptc_weight=float(z["ptc"]))
    x = z["x"]
    got = dict(r_w=res.r_w, r_trace=res.r_trace, matvec=lin.matvec(x),
               rhs=lin.condensed_rhs(res), recover=lin.recover(res, x)[0],
               precond=lin.apply_preconditioner(x))
    for k, v in got.items():
        floor = 1e-12 if k in ("r_w", "r_trace") else 1e-11
        tol = max(floor, 10 * float(z[f"sens_{k}"]))
        assert rel(v, z[k]) <= tol, (k, rel(v, z[k]), tol)
    ints = disc.integrals(fields)
    got_i = np.array([ints[k] for k in KEYS])
    assert np.all(np.abs(got_i - z["integrals"]) <= 1e-12 * np.maximum(1.0, np.abs(z["integrals"])))


class _FirstStep(Exception):
    pass


@pytest.mark.gpu
def test_cfg3_step_through_dt_halving(cuda_ok):
    from paper_2507_22195_b200 import Discretization, DissipationSpec
    from paper_2507_22195_b200.assembly import FieldSet
    from paper_2507_22195_b200.time_march import DIRKIntegrator, NewtonParams

    z = load_golden("cfg3_step_n2")
    gas, tg, mesh = _tgv(2)
    disc = Discretization(mesh, p=3, gas=gas, formulation="entropy",
                          flux=DissipationSpec("kepes"), device="cuda:0")
    f0 = disc.project(tg.initial)
    assert rel(f0.w, z["w0"]) == 0.0 and rel(f0.trace, z["trace0"]) == 0.0
    integ = DIRKIntegrator(disc, params=NewtonParams(max_iters=int(z["max_iters"])))
    got = {}

    def on_step(step, t, flds, reports):
        got.update(t=t, w=flds.w.clone(), trace=flds.trace.clone())
        raise _FirstStep

    with pytest.raises(_FirstStep):
        integ.run(f0, t_final=float(z["dt"]), dt=float(z["dt"]), on_step=on_step)
    assert got["t"] == float(z["t1"])
    newton = np.array([[r["step"], r["stage"], r["newton_iters"]] for r in integ.records])
    assert np.array_equal(newton, z["newton"][:, :3])
    assert rel(got["w"], z["w1"]) <= 1e-10 and rel(got["trace"], z["trace1"]) <= 1e-10
    f1 = FieldSet(got["w"], got["trace"])
    ints = np.array([[disc.integrals(f)[k] for k in KEYS] for f in (f0, f1)])
    want = z["integrals"]
    assert np.all(np.abs(ints - want) <= 1e-12 * np.maximum(1.0, np.abs(want)))
    assert np.sign(ints[1, 0] - ints[0, 0]) == np.sign(want[1, 0] - want[0, 0])


@pytest.mark.gpu
def test_cfg2_step_n8(cuda_ok):
    import math

    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.cases import IsentropicVortex
    from paper_2507_22195_b200.mesh import build_box_macro_mesh
    from paper_2507_22195_b200.time_march import DIRKIntegrator

    z = load_golden("cfg2_step_n8")
    gas = GasModel(1.4)
    vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                          center=(5.0, 5.0), gas=gas)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 8, 1), p=3,
                          gas=gas, formulation="entropy", flux=DissipationSpec("es"),
                          device="cuda:0")
    f0 = disc.project(vx.initial)
    integ = DIRKIntegrator(disc)
    f1, _ = integ.run(f0, t_final=float(z["dt"]), dt=float(z["dt"]))
    newton = np.array([[r["step"], r["stage"], r["newton_iters"]] for r in integ.records])
    assert np.array_equal(newton, z["newton"][:, :3])
    assert rel(f1.w, z["w1"]) <= 1e-10 and rel(f1.trace, z["trace1"]) <= 1e-10
    ints = np.array([[disc.integrals(f)[k] for k in KEYS] for f in (f0, f1)])
    want = z["integrals"]
    assert np.all(np.abs(ints - want) <= 1e-12 * np.maximum(1.0, np.abs(want)))
    assert np.sign(ints[1, 0] - ints[0, 0]) == np.sign(want[1, 0] - want[0, 0])


@pytest.mark.gpu
def test_cfg2_hsweep_first_level(cuda_ok):
    """Config-2 h-refinement study, first level (reference driver.py:570-606
    semantics): n = 8, k = 3, ES, 10 steps of dt = 0.1 to t = 0.1 t_c; the
    L2 error of rho against the exact translated vortex (assembly.py:674-684)
    and the state match the reference; Newton counts identical."""
    import math

    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.cases import IsentropicVortex
    from paper_2507_22195_b200.mesh import build_box_macro_mesh
    from paper_2507_22195_b200.time_march import DIRKIntegrator

    z = load_golden("cfg2_hsweep_n8")
    gas = GasModel(1.4)
    vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                          center=(5.0, 5.0), gas=gas)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 8, 1), p=3,
                          gas=gas, formulation="entropy", flux=DissipationSpec("es"),
                          device="cuda:0")
    f0 = disc.project(vx.initial)
    t_eval = float(z["t_eval"])
    assert abs(disc.l2_error(f0, vx.initial) - float(z["l2_initial"])) <= 1e-12 * float(z["l2_initial"])
    integ = DIRKIntegrator(disc)
    f1, t = integ.run(f0, t_final=t_eval, dt=float(z["dt"]))
    newton = np.array([[r["step"], r["stage"], r["newton_iters"]] for r in integ.records])
    assert np.array_equal(newton, z["newton"][:, :3])
    assert rel(f1.w, z["w1"]) <= 1e-10 and rel(f1.trace, z["trace1"]) <= 1e-10
    err = disc.l2_error(f1, lambda x: vx.state(x, t_eval), component=0)
    assert abs(err - float(z["l2"])) <= 1e-9 * float(z["l2"])

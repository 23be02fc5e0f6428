"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is importable there, not on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Each file holds the seeded inputs and the
reference's outputs for one case, plus the reference's own 1-ulp
self-sensitivity of every output (relative L2 change when w and trace are
perturbed by +-1 ulp), which sets the attainable parity floor
(SURVEY.md finding 11).

Cases
  kat2d_p1_ec      2D two-triangle mesh, p=1, EC flux, seed 13, amp 0.08
                   (the reference's independent hand-assembly KAT,
                   test_assembly.py:488-576)
  sweep_k{1..4}_{flux}
                   config-5 style: 3D unit box, n=(2,2,2), m=1,
                   perturbed-uniform states rho~U[.9,1.1], V~U[-.5,.5],
                   P~U[.9,1.1] per C0 node then per trace node, entropy form;
                   alpha = d00/dt (dt=0.01), offset = -alpha*u_quad,
                   ptc_weight = 1, x ~ N(0,1) with seed+1
  cfg1_*           config 1: vortex on [0,10]^3, n=4, p=2, ES, projected IC;
                   operator outputs at the first stage, the state after one
                   DIRK(3,3) step with dt=0.01, and the integral history of
                   10 steps
  cons_k2_lf       conservative formulation, LF flux (format coverage)
  fs_k2_es         free-stream boundary on a non-periodic box (ghost flux)
  fs_k1_es, fs_k1_kepes, fs_k3_kepes
                   the same at k = 1 and k = 3 (--only-freestream)
  cfg3_*           config 3 (Taylor-Green KEPES k=3): operator at n=4, first
                   accepted step at n=2 through the dt-halving path
  cfg2_step_n8     config 2 at n=8: one DIRK step
  visc_*           viscous operator (gradient unknowns q, level-1 condensation):
                   perturbed states with q = solve_gradient + 0.05 N(0,1) at
                   Re=100, M=0.5; and the config-4 Taylor-Green parameters
                   (Re=1600/M, M=0.1, Pr=0.71) on the projected TGV field
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from macrohdg.assembly import Discretization, FieldSet, FreeStream, StageContext  # noqa: E402
from macrohdg.cases import IsentropicVortex  # noqa: E402
from macrohdg.fluxes import DissipationSpec  # noqa: E402
from macrohdg.cases import TaylorGreen  # noqa: E402
from macrohdg.gas import GasModel, ViscousParams  # noqa: E402
from macrohdg.mesh import build_box_macro_mesh  # noqa: E402
from macrohdg.time_march import DIRKIntegrator, dirk33_tableau  # noqa: E402

GAS = GasModel(1.4)


def perturbed_uniform(disc, seed):
    """Config-5 generator: per C0 node then per trace node."""
    rng = np.random.default_rng(seed)

    def states(n):
        rho = rng.uniform(0.9, 1.1, n)
        vel = rng.uniform(-0.5, 0.5, (n, 3))
        p = rng.uniform(0.9, 1.1, n)
        return GAS.conservative(rho, vel, p)

    E, nc = disc.mesh.n_macros, disc.layout.n_unique
    F, nt = disc.n_faces, disc.layout.n_face_unique
    u_w = states(E * nc).reshape(E, nc, 5)
    u_t = states(F * nt).reshape(F, nt, 5)
    return FieldSet(w=disc.from_conservative(u_w), trace=disc.from_conservative(u_t))


def ulp_perturb(a, rng):
    return a * (1.0 + np.finfo(float).eps * rng.choice([-1.0, 1.0], size=a.shape))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def operator_case(disc, fields, alpha, offset, ptc, x):
    stage = StageContext(alpha=alpha, offset=offset, dt=None)
    res = disc.residuals(fields, stage)
    lin = disc.jacobian(fields, stage, ptc_weight=ptc)
    out = dict(
        r_w=res.r_w, r_trace=res.r_trace,
        matvec=lin.matvec(x), rhs=lin.condensed_rhs(res),
        recover=lin.recover(res, x)[0], precond=lin.apply_preconditioner(x),
        vqs=disc.volume_quad_states(fields),
    )
    return out


def sensitivity(disc, fields, alpha, offset, ptc, x, base, seed=99):
    rng = np.random.default_rng(seed)
    pf = FieldSet(w=ulp_perturb(fields.w, rng), trace=ulp_perturb(fields.trace, rng))
    pert = operator_case(disc, pf, alpha, offset, ptc, x)
    return {f"sens_{k}": rel(pert[k], base[k]) for k in base}


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.1f} kB)")


def meta(disc, flux, formulation, box, n, m, p, periodic=True):
    return dict(box=np.asarray(box, float), n_per_dim=np.asarray(n), m=m, p=p,
                flux=flux, formulation=formulation, periodic=np.asarray(periodic))


def viscous_case(name, disc, fields, alpha, ptc, x, extra):
    """Viscous operator outputs (assembly.py:326-411, 459-549, 772-976,
    1028-1173) on the given fields (with q)."""
    offset = -alpha * disc.volume_quad_states(fields)
    stage = StageContext(alpha=alpha, offset=offset, dt=None)

    def run(f):
        res = disc.residuals(f, stage)
        lin = disc.jacobian(f, stage, ptc_weight=ptc)
        d_w, d_q = lin.recover(res, x)
        return dict(r_w=res.r_w, r_trace=res.r_trace, r_q=res.r_q, matvec=lin.matvec(x),
                    rhs=lin.condensed_rhs(res), recover=d_w, recover_q=d_q,
                    precond=lin.apply_preconditioner(x), vqs=disc.volume_quad_states(f),
                    qgrad=disc.solve_gradient(f))

    out = run(fields)
    rng = np.random.default_rng(99)
    pf = FieldSet(w=ulp_perturb(fields.w, rng), trace=ulp_perturb(fields.trace, rng),
                  q=ulp_perturb(fields.q, rng))
    pert = run(pf)
    sens = {f"sens_{k}": rel(pert[k], out[k]) for k in out}
    save(name, w=fields.w, trace=fields.trace, q=fields.q, offset=offset, alpha=alpha, ptc=ptc,
         x=x, **out, **sens, **extra)


def main_viscous():
    box3 = np.array([[0.0, 1.0]] * 3)
    vp = ViscousParams(reynolds=100.0, mach=0.5)
    for p, flux, form in ((1, "kepes", "entropy"), (2, "kepes", "entropy"), (3, "es", "entropy"),
                          (2, "lf", "conservative")):
        mesh = build_box_macro_mesh(box3, (2, 2, 2), 1)
        disc = Discretization(mesh, p=p, gas=GAS, formulation=form, flux=DissipationSpec(flux),
                              viscosity=vp)
        seed = 2000 + 10 * p
        fields = perturbed_uniform(disc, seed)
        rng = np.random.default_rng(seed + 5)
        fields.q = disc.solve_gradient(fields) + 0.05 * rng.standard_normal(
            fields.w.shape + (3,))
        x = np.random.default_rng(seed + 1).standard_normal(fields.trace.shape)
        viscous_case(f"visc_k{p}_{flux}_{form[:4]}", disc, fields, 40.0, 1.0, x,
                     dict(**meta(disc, flux, form, box3, (2, 2, 2), 1, p), reynolds=100.0,
                          mach=0.5, prandtl=0.72, mu=1.0))
    # Taylor-Green parameters of config 4 (Re 1600 convective -> 16000, Pr 0.71)
    tg = TaylorGreen(mach=0.1, gas=GAS)
    vp = tg.viscous_params(1600.0, prandtl=0.71)
    mesh = build_box_macro_mesh(tg.box, 2, 1)
    disc = Discretization(mesh, p=3, gas=GAS, formulation="entropy",
                          flux=DissipationSpec("kepes"), viscosity=vp)
    fields = disc.project(tg.initial)
    x = np.random.default_rng(31).standard_normal(fields.trace.shape)
    viscous_case("visc_tgv_k3_kepes", disc, fields, 2.29 / 0.57, 1.0, x,
                 dict(**meta(disc, "kepes", "entropy", tg.box, 2, 1, 3),
                      reynolds=vp.reynolds, mach=vp.mach, prandtl=vp.prandtl, mu=vp.mu))


def main_viscous_steps():
    """One DIRK(3,3) step of the viscous Taylor-Green vortex (config-4
    parameters, KEPES) on n=2, p=2, dt = 0.057 t_c."""
    tg = TaylorGreen(mach=0.1, gas=GAS)
    disc = Discretization(build_box_macro_mesh(tg.box, 2, 1), p=2, gas=GAS, formulation="entropy",
                          flux=DissipationSpec("kepes"), viscosity=tg.viscous_params(1600.0, 0.71))
    f0 = disc.project(tg.initial)
    integ = DIRKIntegrator(disc)
    f1, _ = integ.run(f0, t_final=0.57, dt=0.57)
    keys = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")
    newton = np.array([[r["step"], r["stage"], r["newton_iters"], r["fgmres_iters"],
                        r["jacobian_builds"]] for r in integ.records])
    save("visc_tgv_steps", w0=f0.w, trace0=f0.trace, q0=f0.q, w1=f1.w, trace1=f1.trace, q1=f1.q,
         integrals=np.array([[disc.integrals(f)[k] for k in keys] for f in (f0, f1)]),
         dissipation=np.array([disc.kinetic_energy_dissipation(f) for f in (f0, f1)]),
         newton=newton, dt=0.57)


class _FirstStep(Exception):
    pass


def main_cfg3():
    """Config 3 (inviscid Taylor-Green M=0.1, KEPES, k=3):
    cfg3_ops_n4   operator outputs on the projected IC at n=4 (384 macros),
                  alpha = d00/0.57 (the paper's dt), ptc 1, x ~ N(0,1) seed 333
    cfg3_step_n2  the first accepted DIRK(3,3) step at n=2 with dt=2.28 and
                  NewtonParams(max_iters=16): stage 1 needs 17 iterations at
                  2.28, so the step is rejected and retried with dt/2 twice
                  (the integrator's dt-halving path, time_march.py:380-400)"""
    from macrohdg.time_march import NewtonParams

    tg = TaylorGreen(mach=0.1, gas=GAS)
    d00 = dirk33_tableau().d[0, 0]
    mesh = build_box_macro_mesh(tg.box, 4, 1)
    disc = Discretization(mesh, p=3, gas=GAS, formulation="entropy",
                          flux=DissipationSpec("kepes"))
    fields = disc.project(tg.initial)
    alpha = d00 / 0.57
    offset = -alpha * disc.volume_quad_states(fields)
    x = np.random.default_rng(333).standard_normal(fields.trace.shape)
    out = operator_case(disc, fields, alpha, offset, 1.0, x)
    sens = sensitivity(disc, fields, alpha, offset, 1.0, x, out)
    keys = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")
    save("cfg3_ops_n4", w=fields.w, trace=fields.trace, offset=offset, alpha=alpha, ptc=1.0, x=x, **out, **sens,
         integrals=np.array([disc.integrals(fields)[k] for k in keys]),
         **meta(disc, "kepes", "entropy", tg.box, 4, 1, 3))

    mesh = build_box_macro_mesh(tg.box, 2, 1)
    disc = Discretization(mesh, p=3, gas=GAS, formulation="entropy",
                          flux=DissipationSpec("kepes"))
    f0 = disc.project(tg.initial)
    integ = DIRKIntegrator(disc, params=NewtonParams(max_iters=16))
    got = {}

    def on_step(step, t, flds, reports):
        got.update(t=t, w=flds.w.copy(), trace=flds.trace.copy())
        raise _FirstStep

    try:
        integ.run(f0, t_final=2.28, dt=2.28, on_step=on_step)
    except _FirstStep:
        pass
    newton = np.array([[r["step"], r["stage"], r["newton_iters"], r["fgmres_iters"],
                        r["jacobian_builds"]] for r in integ.records])
    save("cfg3_step_n2", w0=f0.w, trace0=f0.trace, w1=got["w"], trace1=got["trace"], t1=got["t"], newton=newton,
         dt=2.28, max_iters=16,
         integrals=np.array([[disc.integrals(f)[k] for k in keys]
                             for f in (f0, FieldSet(got["w"], got["trace"]))]))


def main_cfg2_step():
    """Config 2 (isentropic vortex, ES, k=3) at n=8 (3,072 macros): one
    DIRK(3,3) step with dt=0.01 from the projected IC."""
    vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                          angle=0.0, center=(5.0, 5.0), gas=GAS)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 8, 1), p=3,
                          gas=GAS, formulation="entropy", flux=DissipationSpec("es"))
    f0 = disc.project(vx.initial)
    integ = DIRKIntegrator(disc)
    f1, _ = integ.run(f0, t_final=0.01, dt=0.01)
    keys = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")
    newton = np.array([[r["step"], r["stage"], r["newton_iters"], r["fgmres_iters"],
                        r["jacobian_builds"]] for r in integ.records])
    save("cfg2_step_n8", w1=f1.w, trace1=f1.trace, newton=newton, dt=0.01,
         integrals=np.array([[disc.integrals(f)[k] for k in keys] for f in (f0, f1)]))


def main_entropy():
    """entropy_identity_defect (assembly.py:649-672) on perturbed-uniform
    states (n=(2,2,2)) for es / kepes / ec at p=2, kepes at p=3, and on the
    projected Taylor-Green state (n=2, p=3, kepes)."""
    box3 = np.array([[0.0, 1.0]] * 3)
    out = {}
    for p, flux in ((2, "es"), (2, "kepes"), (2, "ec"), (3, "kepes")):
        disc = Discretization(build_box_macro_mesh(box3, (2, 2, 2), 1), p=p, gas=GAS,
                              formulation="entropy", flux=DissipationSpec(flux))
        f = perturbed_uniform(disc, 3000 + 10 * p)
        lhs, rhs, dfc = disc.entropy_identity_defect(f)
        out[f"k{p}_{flux}"] = (f.w, f.trace, lhs, rhs, dfc)
    tg = TaylorGreen(mach=0.1, gas=GAS)
    disc = Discretization(build_box_macro_mesh(tg.box, 2, 1), p=3, gas=GAS,
                          formulation="entropy", flux=DissipationSpec("kepes"))
    f = disc.project(tg.initial)
    out["tgv_k3_kepes"] = (f.w, f.trace) + tuple(disc.entropy_identity_defect(f))
    arrays = {}
    for k, (w, tr, lhs, rhs, dfc) in out.items():
        arrays.update({f"{k}_w": w, f"{k}_trace": tr, f"{k}_lhs": lhs, f"{k}_rhs": rhs,
                       f"{k}_defect": dfc})
    save("entropy_identity", **arrays)


def main_hsweep():
    """Config-2 h-refinement study, first level (driver.py:570-606 space axis
    semantics on the [0,10]^3 vortex of config 2): n=8, k=3, ES, t_eval =
    0.1 t_c = 1.0, dt0 = t_eval / 10; L2 error of rho against the exact
    translated vortex (assembly.py:674-684) and the final state."""
    vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                          angle=0.0, center=(5.0, 5.0), gas=GAS)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 8, 1), p=3,
                          gas=GAS, formulation="entropy", flux=DissipationSpec("es"))
    f0 = disc.project(vx.initial)
    t_eval = 0.1 * vx.convective_period
    integ = DIRKIntegrator(disc)
    f1, t = integ.run(f0, t_final=t_eval, dt=t_eval / 10.0)
    err = disc.l2_error(f1, lambda x: vx.state(x, t_eval), component=0)
    err0 = disc.l2_error(f0, vx.initial, component=0)
    newton = np.array([[r["step"], r["stage"], r["newton_iters"], r["fgmres_iters"],
                        r["jacobian_builds"]] for r in integ.records])
    save("cfg2_hsweep_n8", w1=f1.w, trace1=f1.trace, l2=err, l2_initial=err0, t_eval=t_eval,
         dt=t_eval / 10.0, newton=newton)


def main_macro():
    """m > 1 macro subdivision: operator outputs on perturbed-
    uniform states, 3D periodic unit box n=(2,1,1) (12 macros), for (m, p) =
    (2,1), (2,2), (2,3), (3,1) with ES (and KEPES at (2,2)); one DIRK(3,3)
    step of the config-1 vortex at m=2, p=2, n=2, dt=0.01."""
    box3 = np.array([[0.0, 1.0]] * 3)
    d00 = dirk33_tableau().d[0, 0]
    for m, p, flux in ((2, 1, "es"), (2, 2, "es"), (2, 2, "kepes"), (2, 3, "es"), (3, 1, "es")):
        mesh = build_box_macro_mesh(box3, (2, 1, 1), m)
        disc = Discretization(mesh, p=p, gas=GAS, formulation="entropy", flux=DissipationSpec(flux))
        seed = 5000 + 100 * m + 10 * p
        fields = perturbed_uniform(disc, seed)
        alpha = d00 / 0.01
        offset = -alpha * disc.volume_quad_states(fields)
        x = np.random.default_rng(seed + 1).standard_normal(fields.trace.shape)
        out = operator_case(disc, fields, alpha, offset, 1.0, x)
        sens = sensitivity(disc, fields, alpha, offset, 1.0, x, out)
        save(f"macro_m{m}_k{p}_{flux}", w=fields.w, trace=fields.trace, offset=offset, alpha=alpha,
             ptc=1.0, x=x, **out, **sens, **meta(disc, flux, "entropy", box3, (2, 1, 1), m, p))
    vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                          angle=0.0, center=(5.0, 5.0), gas=GAS)
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 2, 2), p=2, gas=GAS,
                          formulation="entropy", flux=DissipationSpec("es"))
    f0 = disc.project(vx.initial)
    integ = DIRKIntegrator(disc)
    f1, _ = integ.run(f0, t_final=0.01, dt=0.01)
    keys = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")
    newton = np.array([[r["step"], r["stage"], r["newton_iters"], r["fgmres_iters"],
                        r["jacobian_builds"]] for r in integ.records])
    save("macro_m2_step", w0=f0.w, trace0=f0.trace, w1=f1.w, trace1=f1.trace, newton=newton, dt=0.01,
         integrals=np.array([[disc.integrals(f)[k] for k in keys] for f in (f0, f1)]))


def main_freestream():
    """Free-stream boundary at the other degrees (the far-field flux rows of
    the residual take their own code path per degree on the device)."""
    box3 = np.array([[0.0, 1.0]] * 3)
    uinf = GAS.conservative(1.0, np.array([0.3, -0.2, 0.1]), 0.7)
    for p, flux, seed in ((1, "es", 188), (1, "kepes", 190), (3, "kepes", 192)):
        mesh = build_box_macro_mesh(box3, 2, 1, periodic=(True, False, False))
        disc = Discretization(mesh, p=p, gas=GAS, formulation="entropy",
                              flux=DissipationSpec(flux), boundary=FreeStream(uinf))
        fields = perturbed_uniform(disc, seed)
        x = np.random.default_rng(seed + 1).standard_normal(fields.trace.shape)
        offset = -30.0 * disc.volume_quad_states(fields)
        out = operator_case(disc, fields, 30.0, offset, 1.0, x)
        sens = sensitivity(disc, fields, 30.0, offset, 1.0, x, out)
        save(f"fs_k{p}_{flux}", w=fields.w, trace=fields.trace, offset=offset, alpha=30.0,
             ptc=1.0, x=x, uinf=uinf, **out, **sens,
             **meta(disc, flux, "entropy", box3, 2, 1, p, (True, False, False)))


def main():
    if "--only-freestream" in sys.argv:
        return main_freestream()
    if "--only-macro" in sys.argv:
        return main_macro()
    if "--only-hsweep" in sys.argv:
        return main_hsweep()
    if "--only-entropy" in sys.argv:
        return main_entropy()
    if "--only-cfg3" in sys.argv:
        return main_cfg3()
    if "--only-cfg2-step" in sys.argv:
        return main_cfg2_step()
    if "--only-viscous" in sys.argv:
        return main_viscous()
    if "--only-visc-steps" in sys.argv:
        return main_viscous_steps()
    t0 = time.time()
    tab = dirk33_tableau()
    d00 = tab.d[0, 0]

    # -- 2D KAT --------------------------------------------------------------
    box2 = np.array([[0.0, 1.0]] * 2)
    mesh = build_box_macro_mesh(box2, 1, 1)
    disc = Discretization(mesh, p=1, gas=GAS, formulation="entropy",
                          flux=DissipationSpec("ec"))
    u0 = GAS.conservative(1.0, np.array([0.3, -0.2]), 0.7)
    f = disc.project(lambda x: np.broadcast_to(u0, x.shape[:-1] + (4,)).copy())
    rng = np.random.default_rng(13)
    f.w += 0.08 * rng.standard_normal(f.w.shape)
    f.trace += 0.08 * rng.standard_normal(f.trace.shape)
    res = disc.residuals(f)
    save("kat2d_p1_ec", w=f.w, trace=f.trace, r_w=res.r_w, r_trace=res.r_trace,
         **meta(disc, "ec", "entropy", box2, 1, 1, 1))

    # -- config-5 style sweep ---------------------------------------------------
    box3 = np.array([[0.0, 1.0]] * 3)
    for p in (1, 2, 3, 4):
        fluxes = ("es", "kepes", "ec") if p in (2, 3) else ("es", "kepes")
        for flux in fluxes:
            mesh = build_box_macro_mesh(box3, (2, 2, 2), 1)
            disc = Discretization(mesh, p=p, gas=GAS, formulation="entropy",
                                  flux=DissipationSpec(flux))
            seed = 1000 + 10 * p
            fields = perturbed_uniform(disc, seed)
            dt = 0.01
            alpha = d00 / dt
            offset = -alpha * disc.volume_quad_states(fields)
            x = np.random.default_rng(seed + 1).standard_normal(fields.trace.shape)
            out = operator_case(disc, fields, alpha, offset, 1.0, x)
            sens = sensitivity(disc, fields, alpha, offset, 1.0, x, out)
            save(f"sweep_k{p}_{flux}", w=fields.w, trace=fields.trace, offset=offset,
                 alpha=alpha, ptc=1.0, x=x, **out, **sens,
                 **meta(disc, flux, "entropy", box3, (2, 2, 2), 1, p))

    # -- conservative formulation, LF -------------------------------------------
    mesh = build_box_macro_mesh(box3, (1, 2, 1), 1)
    disc = Discretization(mesh, p=2, gas=GAS, formulation="conservative",
                          flux=DissipationSpec("lf"))
    fields = perturbed_uniform(disc, 77)
    x = np.random.default_rng(78).standard_normal(fields.trace.shape)
    offset = -50.0 * disc.volume_quad_states(fields)
    out = operator_case(disc, fields, 50.0, offset, 0.5, x)
    sens = sensitivity(disc, fields, 50.0, offset, 0.5, x, out)
    save("cons_k2_lf", w=fields.w, trace=fields.trace, offset=offset, alpha=50.0,
         ptc=0.5, x=x, **out, **sens, **meta(disc, "lf", "conservative", box3, (1, 2, 1), 1, 2))

    # -- free-stream boundary ----------------------------------------------------
    mesh = build_box_macro_mesh(box3, 2, 1, periodic=(True, False, False))
    uinf = GAS.conservative(1.0, np.array([0.3, -0.2, 0.1]), 0.7)
    disc = Discretization(mesh, p=2, gas=GAS, formulation="entropy",
                          flux=DissipationSpec("es"), boundary=FreeStream(uinf))
    fields = perturbed_uniform(disc, 88)
    x = np.random.default_rng(89).standard_normal(fields.trace.shape)
    offset = -30.0 * disc.volume_quad_states(fields)
    out = operator_case(disc, fields, 30.0, offset, 1.0, x)
    sens = sensitivity(disc, fields, 30.0, offset, 1.0, x, out)
    save("fs_k2_es", w=fields.w, trace=fields.trace, offset=offset, alpha=30.0,
         ptc=1.0, x=x, uinf=uinf, **out, **sens,
         **meta(disc, "es", "entropy", box3, 2, 1, 2, (True, False, False)))

    # -- config 1 ------------------------------------------------------------
    box = np.array([[0.0, 10.0]] * 3)
    vx = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                          angle=0.0, center=(5.0, 5.0), gas=GAS)
    mesh = build_box_macro_mesh(box, 4, 1)
    disc = Discretization(mesh, p=2, gas=GAS, formulation="entropy",
                          flux=DissipationSpec("es"))
    fields = disc.project(vx.initial)
    dt = 0.01
    alpha = d00 / dt
    offset = -alpha * disc.volume_quad_states(fields)
    x = np.random.default_rng(4242).standard_normal(fields.trace.shape)
    out = operator_case(disc, fields, alpha, offset, 1.0, x)
    sens = sensitivity(disc, fields, alpha, offset, 1.0, x, out)
    save("cfg1_ops", w=fields.w, trace=fields.trace, offset=offset, alpha=alpha,
         ptc=1.0, x=x, node_coords=disc.node_coords, trace_coords=disc.trace_coords,
         **out, **sens, **meta(disc, "es", "entropy", box, 4, 1, 2))

    integ = DIRKIntegrator(disc)
    hist = [disc.integrals(fields)]
    states = {}
    cur = fields

    def on_step(step, t, flds, reports):
        hist.append(disc.integrals(flds))
        if step in (1, 10):
            states[step] = (flds.w.copy(), flds.trace.copy())

    integ.run(cur, t_final=10 * dt, dt=dt, on_step=on_step)
    keys = ("entropy", "thermo_entropy", "kinetic_energy", "mass", "total_energy")
    hist_arr = np.array([[h[k] for k in keys] for h in hist])
    rec = integ.records
    newton = np.array([[r["step"], r["stage"], r["newton_iters"], r["fgmres_iters"],
                        r["jacobian_builds"]] for r in rec])
    save("cfg1_steps", w0=fields.w, trace0=fields.trace, w1=states[1][0],
         trace1=states[1][1], w10=states[10][0], trace10=states[10][1],
         integrals=hist_arr, newton=newton, dt=dt, tableau_d=tab.d, tableau_e=tab.e)
    main_viscous()
    main_viscous_steps()
    main_cfg3()
    main_cfg2_step()
    main_entropy()
    main_macro()
    main_hsweep()
    print(f"done in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    sys.exit(main())

"""CPU timing of the UNMODIFIED reference (macrohdg, installed into
oracle/_ref by oracle/build_ref.sh) on a bounded sample of the bench
workload.  Test / measurement infrastructure: only bench.py's
`--impl reference` arm and its `cpu_baseline` leg run this; it imports
nothing from paper_2507_22195_b200 (no repo .so is loaded).

One "step" is the operator pass the B200 arm times, through the reference's
own public API:
    Discretization.residuals          (reference assembly.py:459-549)
    LinearizedSystem.matvec           (assembly.py:1131-1143)
    LinearizedSystem.apply_preconditioner (assembly.py:1175-1180)
on the state the B200 arm uses (projected initial condition, stage 1 of the
first DIRK(3,3) step: alpha = d00/dt, offset = -alpha u_n, ptc_weight = 1),
on an n_sample^3-cell sub-mesh of the same case.  DoF-applications per step
count the same units as bench.py (residual E*nc*5 + F*nt*5, matvec and
precond F*nt*5 each).

The reference's hot loops are single-threaded Python (per-macro lu_solve,
einsum); "all the host threads it can use" is realised by running one
independent copy of the sample per worker process (OPENBLAS/OMP threads = 1
each), started together; throughput = all workers' DoF-applications / the
slowest worker's timed interval.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def ref_available():
    return os.path.isdir(os.path.join(REF, "macrohdg"))


def _import_ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import macrohdg

    if not os.path.abspath(macrohdg.__file__).startswith(REF):
        raise RuntimeError(f"macrohdg resolved outside oracle/_ref: {macrohdg.__file__}")
    return macrohdg


def build_sample(case, n, p, flux, dt, m=1):
    """Reference objects for the sample: (disc, fields, stage, lin, x, dofs)."""
    import numpy as np

    _import_ref()
    from macrohdg.assembly import Discretization, StageContext
    from macrohdg.cases import IsentropicVortex, TaylorGreen
    from macrohdg.fluxes import DissipationSpec
    from macrohdg.gas import GasModel
    from macrohdg.mesh import build_box_macro_mesh
    from macrohdg.time_march import dirk33_tableau

    gas = GasModel(1.4)
    if case == "tgv":
        ic = TaylorGreen(mach=0.1, gas=gas)
        mesh = build_box_macro_mesh(ic.box, n, m)
    else:
        ic = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                              center=(5.0, 5.0), gas=gas)
        mesh = build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), n, m)
    disc = Discretization(mesh, p=p, gas=gas, formulation="entropy",
                          flux=DissipationSpec(flux))
    fields = disc.project(ic.initial)
    alpha = dirk33_tableau().d[0, 0] / dt
    stage = StageContext(alpha=alpha, offset=-alpha * disc.volume_quad_states(fields), dt=dt)
    lin = disc.jacobian(fields, stage, ptc_weight=1.0)
    x = np.random.default_rng(1).standard_normal(lin.trace_shape)
    E = mesh.n_macros
    F, nt = lin.trace_shape[0], lin.trace_shape[1]
    nc = fields.w.shape[1]
    dofs = (E * nc * 5 + F * nt * 5) + 2 * F * nt * 5
    return disc, fields, stage, lin, x, dofs, E


def _worker(args):
    case, n, p, flux, dt, m, warmup, steps, budget_s, barrier = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(1)
    except Exception:   # threadpoolctl absent: env vars above still apply to new pools
        limiter = None
    disc, fields, stage, lin, x, dofs, E = build_sample(case, n, p, flux, dt, m)

    def step():
        disc.residuals(fields, stage)
        lin.matvec(x)
        lin.apply_preconditioner(x)

    for _ in range(warmup):
        step()
    if barrier is not None:
        barrier.wait()
    t0 = time.perf_counter()
    done = 0
    while True:
        step()
        done += 1
        el = time.perf_counter() - t0
        if (steps is not None and done >= steps) or (steps is None and el >= budget_s):
            break
    if limiter is not None:
        limiter.unregister() if hasattr(limiter, "unregister") else None
    return dict(steps=done, seconds=el, dofs=dofs, macros=E)


def time_reference(case="tgv", n=4, p=3, flux="kepes", dt=0.57, workers=1, warmup=1,
                   steps=None, budget_s=10.0, m=1):
    """Run `workers` concurrent copies; returns the throughput summary."""
    if not ref_available():
        raise RuntimeError("oracle/_ref missing: run oracle/build_ref.sh in the build container")
    if workers <= 1:
        r = _worker((case, n, p, flux, dt, m, warmup, steps, budget_s, None))
        res = [r]
    else:
        ctx = mp.get_context("spawn")
        mgr = ctx.Manager()
        barrier = mgr.Barrier(workers)
        with ctx.Pool(workers) as pool:
            res = pool.map(_worker, [(case, n, p, flux, dt, m, warmup, steps, budget_s, barrier)] *
                           workers)
    total = sum(r["dofs"] * r["steps"] for r in res)
    span = max(r["seconds"] for r in res)
    steps_each = [r["steps"] for r in res]
    return dict(value=total / span, unit="DoF-applications/s", cores=workers, kind="reference",
                seconds_per_step=span / min(steps_each), steps=steps_each, span_s=span,
                sample=(f"unmodified reference macrohdg (oracle/_ref) residual+matvec+precond, "
                        f"{'Taylor-Green M=0.1' if case == 'tgv' else 'isentropic vortex'} "
                        f"n={n} sub-mesh ({res[0]['macros']} macros) k={p} m={m} {flux}, "
                        f"{workers} concurrent single-threaded copies, "
                        f"{sum(steps_each)} steps over {span:.1f} s"))


if __name__ == "__main__":
    import json

    print(json.dumps(time_reference(n=int(sys.argv[1]) if len(sys.argv) > 1 else 2,
                                    workers=int(sys.argv[2]) if len(sys.argv) > 2 else 1,
                                    budget_s=3.0)))

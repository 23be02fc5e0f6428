"""GPU parity: the CUDA operator (through the C ABI) against the reference's
golden vectors and the pinned CPU oracle on identical seeded inputs.

Tolerances (relative L2), per SURVEY.md 8c / finding 11:
  residual                     <= max(1e-12, 10 x reference 1-ulp sensitivity)
  matvec / rhs / recover / precond
                               <= max(1e-11, 10 x reference 1-ulp sensitivity)
  volume quadrature states     <= 1e-14
"""

import numpy as np
import pytest

from helpers import golden_mesh, load_golden, rel

pytestmark = pytest.mark.gpu

CASES = ["sweep_k1_es", "sweep_k1_kepes", "sweep_k2_es", "sweep_k2_kepes", "sweep_k2_ec",
         "sweep_k3_es", "sweep_k3_kepes", "sweep_k3_ec", "sweep_k4_es", "sweep_k4_kepes",
         "cons_k2_lf", "fs_k2_es", "fs_k1_es", "fs_k1_kepes", "fs_k3_kepes", "cfg1_ops"]


def make_disc(z):
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.assembly import FreeStream

    bd = FreeStream(z["uinf"]) if "uinf" in z else None
    return Discretization(golden_mesh(z), p=int(z["p"]), gas=GasModel(1.4),
                          formulation=str(z["formulation"]),
                          flux=DissipationSpec(str(z["flux"])), boundary=bd, device="cuda:0")


def tol(z, key, floor):
    return max(floor, 10.0 * float(z.get(f"sens_{key}", 0.0)))


@pytest.fixture(scope="module", params=CASES)
def case(request, cuda_ok):
    from paper_2507_22195_b200 import StageContext
    from paper_2507_22195_b200.assembly import FieldSet

    z = load_golden(request.param)
    disc = make_disc(z)
    fields = FieldSet(z["w"], z["trace"])
    stage = StageContext(alpha=float(z["alpha"]), offset=z["offset"])
    res = disc.residuals(fields, stage)
    lin = disc.jacobian(fields, stage, ptc_weight=float(z["ptc"]))
    return request.param, z, disc, fields, stage, res, lin


def test_residual(case):
    name, z, disc, fields, stage, res, lin = case
    assert rel(res.r_w, z["r_w"]) <= tol(z, "r_w", 1e-12), name
    assert rel(res.r_trace, z["r_trace"]) <= tol(z, "r_trace", 1e-12), name


def test_matvec(case):
    name, z, disc, fields, stage, res, lin = case
    assert rel(lin.matvec(z["x"]), z["matvec"]) <= tol(z, "matvec", 1e-11), name


def test_condensed_rhs(case):
    name, z, disc, fields, stage, res, lin = case
    assert rel(lin.condensed_rhs(res), z["rhs"]) <= tol(z, "rhs", 1e-11), name


def test_recover(case):
    name, z, disc, fields, stage, res, lin = case
    d_w, d_q = lin.recover(res, z["x"])
    assert d_q is None
    assert rel(d_w, z["recover"]) <= tol(z, "recover", 1e-11), name


def test_preconditioner(case):
    name, z, disc, fields, stage, res, lin = case
    assert rel(lin.apply_preconditioner(z["x"]), z["precond"]) <= tol(z, "precond", 1e-11), name


def test_volume_quad_states(case):
    name, z, disc, fields, stage, res, lin = case
    assert rel(disc.volume_quad_states(fields), z["vqs"]) <= 1e-14, name


def test_deterministic(case):
    name, z, disc, fields, stage, res, lin = case
    r2 = disc.residuals(fields, stage)
    assert bool((r2.r_w == res.r_w).all()) and bool((r2.r_trace == res.r_trace).all())
    y1, y2 = lin.matvec(z["x"]), lin.matvec(z["x"])
    assert bool((y1 == y2).all())


def test_kepes_vs_oracle_fresh_seed(cuda_ok):
    """Device vs the pinned oracle on a fresh seed (not in any golden)."""
    from oracle.hdg_oracle import OracleHDG
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel, StageContext
    from paper_2507_22195_b200.assembly import FieldSet
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    mesh = build_box_macro_mesh(np.array([[0.0, 2.0]] * 3), (2, 1, 2), 1)
    disc = Discretization(mesh, p=3, gas=gas, flux=DissipationSpec("kepes"), device="cuda:0")
    rng = np.random.default_rng(31337)
    E, nc, F, nt = mesh.n_macros, disc.layout.n_unique, disc.n_faces, disc.layout.n_face_unique

    def st(n):
        return gas.entropy_vars(gas.conservative(rng.uniform(0.9, 1.1, n),
                                                 rng.uniform(-0.5, 0.5, (n, 3)),
                                                 rng.uniform(0.9, 1.1, n)))

    w, tr = st(E * nc).reshape(E, nc, 5), st(F * nt).reshape(F, nt, 5)
    ora = OracleHDG(disc.tables, flux="kepes")
    off = -100.0 * ora.volume_quad_states(w)
    res = disc.residuals(FieldSet(w, tr), StageContext(100.0, off))
    rw, rt = ora.residuals(w, tr, 100.0, off)
    assert rel(res.r_w, rw) <= 1e-12 and rel(res.r_trace, rt) <= 1e-12
    lin = disc.jacobian(FieldSet(w, tr), StageContext(100.0, off), ptc_weight=2.0)
    olin = ora.linearize(w, tr, 100.0, 2.0)
    x = rng.standard_normal(tr.shape)
    assert rel(lin.matvec(x), olin.matvec(x)) <= 1e-10
    assert rel(lin.apply_preconditioner(x), olin.apply_preconditioner(x)) <= 1e-10


def test_freestream_preserved(cuda_ok):
    """Uniform state: residual <= 1e-12 (test_assembly.py:83-106 analogue)."""
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel

    gas = GasModel(1.4)
    mesh = __import__("paper_2507_22195_b200.mesh", fromlist=["x"]).build_box_macro_mesh(
        np.array([[0.0, 1.0]] * 3), 2, 1)
    u0 = gas.conservative(1.0, np.array([0.3, -0.2, 0.1]), 0.7)
    for flux in ("lf", "ec", "es", "kepes"):
        for form in ("entropy", "conservative"):
            disc = Discretization(mesh, p=2, gas=gas, formulation=form,
                                  flux=DissipationSpec(flux), device="cuda:0")
            f = disc.project(lambda x: np.broadcast_to(u0, x.shape[:-1] + (5,)).copy())
            assert disc.residuals(f).max_abs() <= 1e-12, (flux, form)


def test_admissibility_errors(cuda_ok):
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.errors import NonAdmissibleState
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), 1, 1)
    u0 = gas.conservative(1.0, np.array([0.3, -0.2, 0.1]), 0.7)
    disc = Discretization(mesh, p=1, gas=gas, formulation="conservative",
                          flux=DissipationSpec("es"), device="cuda:0")
    f = disc.project(lambda x: np.broadcast_to(u0, x.shape[:-1] + (5,)).copy())
    f.w[0, 0, -1] = -9.0
    with pytest.raises(NonAdmissibleState) as exc:
        disc.residuals(f)
    assert "volume" in str(exc.value) and exc.value.where
    f = disc.project(lambda x: np.broadcast_to(u0, x.shape[:-1] + (5,)).copy())
    f.trace[0, 0, -1] = -9.0
    with pytest.raises(NonAdmissibleState) as exc:
        disc.residuals(f)
    assert "trace" in str(exc.value)


def test_integrals_vs_oracle(cuda_ok):
    from oracle.hdg_oracle import OracleHDG

    z = load_golden("cfg1_ops")
    disc = make_disc(z)
    from paper_2507_22195_b200.assembly import FieldSet

    got = disc.integrals(FieldSet(z["w"], z["trace"]))
    want = OracleHDG(disc.tables, flux="es").integrals(z["w"])
    for k in want:
        assert abs(got[k] - want[k]) <= 1e-12 * max(1.0, abs(want[k])), k


def test_entropy_state_error(cuda_ok):
    """v5 >= 0 in the entropy formulation -> NonAdmissibleEntropyState (a
    NonAdmissibleState) located in the volume, as the reference's
    from_entropy raises it (gas.py:163-168)."""
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.errors import NonAdmissibleEntropyState, NonAdmissibleState
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), 1, 1)
    u0 = gas.conservative(1.0, np.array([0.3, -0.2, 0.1]), 0.7)
    disc = Discretization(mesh, p=2, gas=gas, formulation="entropy",
                          flux=DissipationSpec("es"), device="cuda:0")
    f = disc.project(lambda x: np.broadcast_to(u0, x.shape[:-1] + (5,)).copy())
    w = f.w.cpu().numpy() if hasattr(f.w, "cpu") else np.array(f.w)
    w[2, :, 4] = 0.5   # every volume point of macro 2: the volume pass fails first
    f.w = w
    with pytest.raises(NonAdmissibleEntropyState) as exc:
        disc.residuals(f)
    assert isinstance(exc.value, NonAdmissibleState)
    assert "volume" in str(exc.value) and "macro 2" in str(exc.value)


def test_singular_local_matrix_names_the_macro(cuda_ok):
    """A non-finite state in one macro makes its condensed block singular:
    SingularLocalMatrix(macro=e) for that macro (assembly.py:718-733)."""
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel, StageContext
    from paper_2507_22195_b200.errors import SingularLocalMatrix
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    mesh = build_box_macro_mesh(np.array([[0.0, 1.0]] * 3), 2, 1)
    u0 = gas.conservative(1.0, np.array([0.3, -0.2, 0.1]), 0.7)
    disc = Discretization(mesh, p=3, gas=gas, formulation="entropy",
                          flux=DissipationSpec("es"), device="cuda:0")
    f = disc.project(lambda x: np.broadcast_to(u0, x.shape[:-1] + (5,)).copy())
    w = f.w.cpu().numpy() if hasattr(f.w, "cpu") else np.array(f.w)
    w[5, :, 0] = np.nan
    f.w = w
    with pytest.raises(SingularLocalMatrix) as exc:
        disc.jacobian(f, StageContext(alpha=10.0, offset=None), ptc_weight=1.0)
    assert exc.value.macro == 5

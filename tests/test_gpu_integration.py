"""INTEGRATION.md claim, checked: the UNMODIFIED reference time march
(macrohdg.time_march from oracle/_ref, installed by oracle/build_ref.sh)
drives this package's device Discretization.  The reference's
newton_solve / advance_step only duck-type `disc`; its solve_condensed is
patched to the device one, the injection point the reference's own tests
use (test_time_march.py:246-262).  One config-1 step must reproduce the
reference's converged state (tests/golden/cfg1_steps.npz) and Newton
counts.  The reference is test infrastructure here, as in bench.py's
reference arm; skipped when oracle/_ref is absent."""

import os
import sys

import numpy as np
import pytest

from helpers import ROOT, load_golden, rel

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "oracle", "_ref")


@pytest.fixture
def ref_time_march(monkeypatch):
    if not os.path.isdir(os.path.join(REF, "macrohdg")):
        pytest.skip("oracle/_ref not built (oracle/build_ref.sh)")
    monkeypatch.syspath_prepend(REF)
    import macrohdg.time_march as tm

    assert os.path.abspath(tm.__file__).startswith(REF)
    from paper_2507_22195_b200 import solver

    monkeypatch.setattr(tm, "solve_condensed", solver.solve_condensed)
    yield tm
    for name in [m for m in sys.modules if m == "macrohdg" or m.startswith("macrohdg.")]:
        sys.modules.pop(name)


def test_reference_advance_step_drives_device_disc(cuda_ok, ref_time_march):
    from paper_2507_22195_b200 import Discretization, DissipationSpec, GasModel
    from paper_2507_22195_b200.assembly import FieldSet
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    tm = ref_time_march
    z = load_golden("cfg1_steps")
    disc = Discretization(build_box_macro_mesh(np.array([[0.0, 10.0]] * 3), 4, 1), p=2,
                          gas=GasModel(1.4), formulation="entropy", flux=DissipationSpec("es"),
                          device="cuda:0")
    fields = FieldSet(disc._dev(z["w0"]), disc._dev(z["trace0"]))
    out, reports = tm.advance_step(disc, fields, 0.0, float(z["dt"]), cache=tm.JacobianCache())
    assert rel(out.w, z["w1"]) <= 1e-10 and rel(out.trace, z["trace1"]) <= 1e-10
    want = z["newton"][z["newton"][:, 0] == 1][:, 2]
    assert [r.newton_iters for r in reports] == list(want)

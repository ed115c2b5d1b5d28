"""Device parity, bit-flip spin registers (QOC_KIND_BITFLIP, BASELINE config 3): the sm_100a
Neumann/Jacobi Cayley kernels vs the CPU oracle (structured arithmetic, itself pinned against
the dense-LU reference arithmetic in test_oracle_kats.py)."""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import problems
from tests import oracle_api as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


# nspins 5..12 cover every amplitudes-per-thread instantiation (E = 1, 2, 4, 8, 16)
@pytest.mark.parametrize("nspins", [5, 8, 9, 10, 11, 12])
def test_propagate_and_gradient(ctx, nspins):
    w = problems.ising10(nspins=nspins, steps=24, T=0.18)
    u = w.u0
    fin = I.propagate_final(w.problem, u, ctx)
    ref = O.propagate_final(w.problem, u, O.STRUCTURED)
    assert np.max(np.abs(fin - ref)) < 1e-13
    for form in ("overlap", "tracking"):
        v, g = I.objective_gradient(w.problem, u, form, ctx=ctx)
        vr, gr = O.objective_gradient(w.problem, u, form, arith=O.STRUCTURED)
        assert abs(v[0] - vr[0]) < 1e-13
        assert np.max(np.abs(g - gr)) < 1e-13


def test_matches_dense_lu_reference_arithmetic(ctx):
    w = problems.ising10(nspins=6, steps=30, T=0.3)
    fin = I.propagate_final(w.problem, w.u0, ctx)
    ref = O.propagate_final(w.problem, w.u0, O.REFERENCE)  # Eigen-style dense partial-pivot LU
    assert np.max(np.abs(fin - ref)) < 1e-13


@pytest.mark.parametrize("parts,plan", [(1, "assembled"), (4, "assembled"), (7, "direct"), (16, "direct")])
def test_run_ism_small_register(ctx, parts, plan):
    w = problems.ising10(nspins=6, steps=64, T=0.5, iterations=4, subintervals=parts, rho=2.0)
    w.config.plan = plan
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0]
    assert rel(g.control, r.control) < 1e-11
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-11
    for a, b in zip(g.record.iterations[1:], r.record.iterations[1:]):
        assert abs(a.error - b.error) < 1e-10 * max(1.0, abs(b.error))


FIXTURES = __import__("pathlib").Path(__file__).parent / "golden"


def compare_run(g, fx, tag, ctl_tol=1e-9, obj_tol=1e-10, u0=None, upd_tol=1e-5, tv_tol=None):
    assert rel(g.control, fx[f"{tag}_control"]) < ctl_tol
    if u0 is not None:  # the update itself (config 3's gradient is ~1e-9: u moves ~1e-8 in 20 iterations)
        du_ref = fx[f"{tag}_control"] - np.asarray(u0)
        assert np.max(np.abs(du_ref)) > 0
        assert rel(g.control - np.asarray(u0), du_ref) < upd_tol
    obj = fx[f"{tag}_objective"]
    assert len(g.record.iterations) == len(obj)
    assert np.max(np.abs(g.record.objectives() - obj)) < obj_tol
    err = np.array([np.nan if it.error is None else it.error for it in g.record.iterations])
    ok = np.isfinite(fx[f"{tag}_error"])
    assert np.array_equal(np.isfinite(err), ok)
    assert np.max(np.abs(err[ok] - fx[f"{tag}_error"][ok]) / np.maximum(1.0, np.abs(fx[f"{tag}_error"][ok]))) < 1e-9
    tv = np.array([it.task_values for it in g.record.iterations])
    assert np.max(np.abs(tv - fx[f"{tag}_task_values"])) < (obj_tol if tv_tol is None else tv_tol)


@pytest.mark.slow
@pytest.mark.parametrize("tag", ["literal", "fast"])
def test_ising10_config3_iterations(ctx, tag):
    # BASELINE config 3 at full size (d = 1024, K = 4000, L = 256) for its timing count of 20
    # outer iterations at rho = 0.1 and rho = 0.1/dt, against the oracle's frozen outputs
    # (tests/golden/make_baseline_fixtures.py)
    fx = np.load(FIXTURES / "config3_full.npz")
    w = problems.ising10(iterations=20)
    w.solver.step_size = float(fx[f"{tag}_rho"])
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    compare_run(g, fx, tag, u0=w.u0)

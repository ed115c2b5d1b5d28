"""Device parity, tridiagonal operators (BASELINE config 2, the rigid rotor)."""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import models as M
from paper_1603_01237_b200 import problems
from tests import oracle_api as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def tri_fixture(seed, d=7, K=16, C=2, quad=False):
    rng = np.random.default_rng(seed)
    nops = 1 + C * (2 if quad else 1)
    diag = rng.standard_normal((nops, d))
    sub = rng.standard_normal((nops, d - 1)) + 1j * rng.standard_normal((nops, d - 1))
    model = M.TridiagonalModel(diag, sub, C, quad)
    ini = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    tgt = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    p = I.ControlProblem(model, I.TimeGrid.over(0, 1.0, K), ini / np.linalg.norm(ini), tgt / np.linalg.norm(tgt),
                         rng.uniform(0, 0.1, K))
    return p, rng.uniform(-0.8, 0.8, (C, K))


@pytest.mark.parametrize("quad", [False, True])
@pytest.mark.parametrize("d", [2, 7, 21, 30])
def test_tridiag_helpers(ctx, quad, d):
    p, u = tri_fixture(d + 10 * quad, d=d, quad=quad)
    dense = I.ControlProblem(p.model.to_dense(), p.grid, p.initial, p.target, p.penalty)
    fin = I.propagate_final(p, u, ctx)
    assert np.max(np.abs(fin - O.propagate_final(dense, u, O.REFERENCE))) < 1e-13
    for form in ("overlap", "tracking"):
        v, g = I.objective_gradient(p, u, form, ctx=ctx)
        vr, gr = O.objective_gradient(dense, u, form, arith=O.REFERENCE)
        assert abs(v[0] - vr[0]) < 1e-13 and np.max(np.abs(g - gr)) < 1e-13
    Mt = I.assemble_propagator(p, u, ctx)
    assert np.max(np.abs(Mt - O.assemble_propagator(dense, u, O.REFERENCE))) < 1e-13


@pytest.mark.parametrize("parts", [1, 3, 4])
@pytest.mark.parametrize("variant,plan", [("interpolated", "assembled"), ("interpolated", "direct"),
                                          ("split", "assembled")])
def test_tridiag_run(ctx, parts, variant, plan):
    p, u = tri_fixture(77)
    cfg = I.IsmConfig(subintervals=parts, max_outer=6, eta=0.0, variant=variant, plan=plan)
    sv = I.SolverSpec(step_size=0.4)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv, O.STRUCTURED)[0]
    assert np.max(np.abs(g.control - r.control)) < 1e-12
    assert np.nanmax(np.abs(g.record.objectives() - r.record.objectives())) < 1e-12


@pytest.mark.parametrize("L", [1, 8, 32, 128])
def test_rotor21_config(ctx, L):
    w = problems.rotor21(subintervals=L, iterations=10, rho=100.0)
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0]
    assert rel(g.control, r.control) < 1e-9
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-10


@pytest.mark.slow
@pytest.mark.parametrize("rho", [0.1, 100.0])  # literal rho and rho = 0.1/dt
def test_rotor21_config_200_iterations(ctx, rho):
    # north_star parity bar at BASELINE size: L = 128 (32 x 157 + 96 x 156), 200 iterations
    w = problems.rotor21(subintervals=128, iterations=200, rho=rho)
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0]
    assert rel(g.control, r.control) < 1e-9
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-10

"""The restated oracle pinned to the REFERENCE ITSELF.

oracle/_ref/libqocref.so is /root/reference/proj/core's own run_ism and everything under it
(ism, objective, optimizers, propagation, controls, linalg, models, runtime .cpp, unmodified),
compiled by `make -C oracle ref` against the Eigen-subset shim oracle/eigen_shim.  These CPU
tests run both on the same packed problems -- every operator kind, both variants, both plans,
L in {1, 2, 4, 8}, the inner-iteration count, the naive split adjoint, the abort path, and the
full 200-iteration BASELINE config 1 -- and require agreement to rounding (the shim's LU and the
oracle's LU differ only in summation order).  The reference's Decomposition::uniform is kept on
its side, so every case uses K % L == 0 (ism.cpp:234).

Skipped where /root/reference is absent (the GPU box).
"""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import problems
from tests import oracle_api as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference tree not present")


def compare(r, o, ctl_abs=1e-12, obj_abs=1e-12):
    scale = max(1.0, float(np.max(np.abs(r.control))))
    assert np.max(np.abs(r.control - o.control)) <= ctl_abs * scale
    assert len(r.record.iterations) == len(o.record.iterations)
    assert r.record.aborted == o.record.aborted and r.record.abort_reason == o.record.abort_reason
    for a, b in zip(r.record.iterations, o.record.iterations):
        assert a.iteration == b.iteration
        if np.isfinite(a.objective) or np.isfinite(b.objective):
            assert abs(a.objective - b.objective) <= obj_abs
        assert (a.error is None) == (b.error is None)
        if a.error is not None:
            assert abs(a.error - b.error) <= 1e-11 * max(1.0, abs(a.error))
        assert (a.exact_objective is None) == (b.exact_objective is None)
        if a.exact_objective is not None:
            assert abs(a.exact_objective - b.exact_objective) <= obj_abs
        ta, tb = np.asarray(a.task_values, float), np.asarray(b.task_values, float)
        assert np.array_equal(np.isfinite(ta), np.isfinite(tb))
        ok = np.isfinite(ta)
        if ok.any():
            assert np.max(np.abs(ta[ok] - tb[ok])) <= obj_abs


@pytest.mark.parametrize("dim,channels,quad", [(2, 1, False), (4, 2, True), (7, 2, False), (5, 3, True)])
@pytest.mark.parametrize("parts", [1, 2, 4, 8])
@pytest.mark.parametrize("variant,plan", [("interpolated", "assembled"), ("interpolated", "direct"),
                                          ("split", "assembled"), ("split", "direct")])
def test_dense_runs(dim, channels, quad, parts, variant, plan):
    p, u = O.dense_fixture(5000 + dim + 10 * channels, dim=dim, steps=16, channels=channels, quadratic=quad,
                           random_penalty=True)
    cfg = I.IsmConfig(subintervals=parts, max_outer=5, eta=0.0, variant=variant, plan=plan,
                      log_exact_objective=(variant == "split"), partition="uniform")
    sv = I.SolverSpec(step_size=0.5)
    compare(O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv, O.REFERENCE)[0])


@pytest.mark.parametrize("inner", [0, 2])
def test_inner_iterations(inner):
    p, u = O.dense_fixture(5100, dim=4, steps=24, random_penalty=True)
    cfg = I.IsmConfig(subintervals=4, max_outer=4, eta=0.0, partition="uniform")
    sv = I.SolverSpec(step_size=0.4, inner_iterations=inner)
    compare(O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv, O.REFERENCE)[0])


def test_eta_stop_and_abort_path():
    p, u = O.dense_fixture(2800)
    cfg = I.IsmConfig(subintervals=2, max_outer=50, eta=1e9, partition="uniform")
    compare(O.ref_ism_run(p, u, cfg, I.SolverSpec(step_size=0.1))[0],
            O.ism_run(p, u, cfg, I.SolverSpec(step_size=0.1), O.REFERENCE)[0])
    p, u = O.dense_fixture(2700, random_penalty=True)
    cfg = I.IsmConfig(subintervals=4, max_outer=40, eta=0.0, partition="uniform")
    sv = I.SolverSpec(step_size=1e300)
    r = O.ref_ism_run(p, u, cfg, sv)[0]
    o = O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    assert r.record.aborted and o.record.aborted and r.record.abort_reason == o.record.abort_reason
    assert len(r.record.iterations) == len(o.record.iterations)
    fin = np.isfinite(r.control)
    assert np.array_equal(fin, np.isfinite(o.control))
    assert np.allclose(r.control[fin], o.control[fin], rtol=1e-12, atol=0)


@pytest.mark.parametrize("rho", [0.1, 10.0])
def test_config1_spin2_full_run(rho):
    # BASELINE config 1 exactly (K = 1000, L = 8, 200 outer iterations) through the reference
    w = problems.spin2(rho=rho)
    r = O.ref_ism_run(w.problem, w.u0, w.config, w.solver)[0]
    o = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0]
    compare(r, o, ctl_abs=1e-12, obj_abs=1e-12)


def test_rotor_tridiagonal_kind():
    # config-2 physics, K = 2000, L = 16: the reference builds the rotor as a dense model; the
    # oracle's structured (Thomas) and dense-LU arithmetic both match it
    w = problems.rotor21(subintervals=16, iterations=4, rho=100.0)
    p = w.problem
    K = 2000
    w.problem = I.ControlProblem(p.model, I.TimeGrid(0.0, p.grid.dt, K), p.initial, p.target, np.zeros(K))
    w.u0 = np.asarray(w.u0)[:, :K]
    w.config.partition = "uniform"
    r = O.ref_ism_run(w.problem, w.u0, w.config, w.solver)[0]
    compare(r, O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0], ctl_abs=1e-11, obj_abs=1e-11)
    compare(r, O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0], ctl_abs=1e-11, obj_abs=1e-11)


@pytest.mark.parametrize("plan", ["assembled", "direct"])
def test_spin_register_bitflip_kind(plan):
    # config-3 kind on 6 spins (d = 64): the reference propagates the dense expansion with LU;
    # the oracle's structured Neumann/Jacobi solve matches it
    w = problems.ising10(nspins=6, steps=64, T=0.5, iterations=4, subintervals=8, rho=2.0)
    w.config.plan = plan
    w.config.partition = "uniform"
    r = O.ref_ism_run(w.problem, w.u0, w.config, w.solver)[0]
    compare(r, O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0], ctl_abs=1e-11, obj_abs=1e-11)


def test_kat8_condensate_preset_by_the_reference():
    # acceptance_main.cpp:439-485 run by the reference itself: 10 iterations, N = 4, rho = 0.1,
    # exact payoff >= -0.742728295 (1e-6) and strictly increasing; the oracle agrees with it
    w = problems.condensate_preset(subintervals=4, iterations=10)
    r = O.ref_ism_run(w.problem, w.u0, w.config, w.solver)[0]
    pay = [it.exact_objective for it in r.record.iterations[1:]]
    assert all(b > a for a, b in zip(pay, pay[1:]))
    assert pay[-1] >= -0.742728295 - 1e-6
    compare(r, O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0], ctl_abs=1e-11, obj_abs=1e-11)


@pytest.mark.parametrize("naive", [False, True])
def test_lattice_condensate_split(naive):
    # the config-4 potential (harmonic + cos^2 lattice) on 64 points through the reference's
    # split-step kernels behind its plugin interface
    from tests.test_gpu_strang import lattice_problem
    p, u = lattice_problem(64, steps=32, T=0.1)
    cfg = I.IsmConfig(subintervals=4, max_outer=5, eta=0.0, variant="split", log_exact_objective=True,
                      partition="uniform")
    sv = I.SolverSpec(step_size=0.3, naive_nonlinear_adjoint=naive)
    compare(O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv, O.STRUCTURED)[0], ctl_abs=1e-11,
            obj_abs=1e-11)


def test_config5_batch_problems():
    # config-5 problems (d = 16, K = 2000) with L = 125 (uniform 16-step parts), 2 iterations each
    w = problems.batch4096(batch=3, iterations=2, subintervals=125)
    w.solver.step_size = w.rho_fast
    w.config.partition = "uniform"
    for r, o in zip(O.ref_ism_run(w.problem, w.u0, w.config, w.solver),
                    O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)):
        compare(r, o, ctl_abs=1e-12, obj_abs=1e-12)


def test_integration_shim_compiles():
    # INTEGRATION.md's reference-side translation unit, compiled against the reference headers
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    subprocess.run(["make", "-s", "-C", str(root / "integration"), "_build/ism_gpu.o"], check=True)
    assert (root / "integration" / "_build" / "ism_gpu.o").exists()


@pytest.mark.parametrize("plan", ["assembled", "direct"])
@pytest.mark.parametrize("parts", [1, 4])
def test_density_matrix_spins_preset(plan, parts):
    # the reference's `spins` preset (density-matrix conjugation kind, models.cpp:320-347,
    # propagation.cpp:92-129, objective.cpp:61-71), quick size: 3 spins, 2^10 steps, rho = 1e4
    w = problems.spins_preset(quick=True, subintervals=parts, iterations=5)
    w.config.plan = plan
    w.config.partition = "uniform"
    compare(O.ref_ism_run(w.problem, w.u0, w.config, w.solver)[0],
            O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0], ctl_abs=1e-12, obj_abs=1e-12)


def test_density_matrix_five_spins():
    # the paper's 5-spin chain (d = 32, ten x/y channels) on a shortened grid
    w = problems.spins_preset(quick=False, subintervals=4, iterations=3, steps=128)
    w.config.partition = "uniform"
    compare(O.ref_ism_run(w.problem, w.u0, w.config, w.solver)[0],
            O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0], ctl_abs=1e-11, obj_abs=1e-11)


# ---- the other two inner solvers (optimizers.cpp:109-259), SURVEY §8(f) ranks 3-4 -------------
def _events(run):
    return [list(it.events) for it in run.record.iterations]


@pytest.mark.parametrize("dim,quad", [(2, False), (3, True), (6, False)])
@pytest.mark.parametrize("parts", [1, 4])
@pytest.mark.parametrize("variant", ["interpolated", "split"])
def test_monotonic_sweep(dim, quad, parts, variant):
    p, u = O.dense_fixture(6000 + dim, dim=dim, steps=24, channels=1, quadratic=quad, alpha=0.15)
    cfg = I.IsmConfig(subintervals=parts, max_outer=6, eta=0.0, variant=variant, partition="uniform")
    sv = I.SolverSpec(kind="monotonic", inner_iterations=1)
    r, o = O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    compare(r, o, ctl_abs=1e-11, obj_abs=1e-11)
    assert _events(r) == _events(o)  # guard rejections per task, as the reference words them


def test_monotonic_sweep_moves_the_control_and_rejections_are_counted():
    p, u = O.dense_fixture(1002, dim=2, steps=24, channels=1, alpha=0.15)  # optimizers_test.cpp:52-76
    cfg = I.IsmConfig(subintervals=4, max_outer=3, eta=0.0, partition="uniform")
    sv = I.SolverSpec(kind="monotonic")
    r, o = O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    assert np.max(np.abs(o.control - np.asarray(u))) > 1e-6
    assert _events(r) == _events(o)


@pytest.mark.parametrize("kw,msg", [
    (dict(channels=2, alpha=0.1), "single control channel"),
    (dict(channels=1, alpha=0.0), "strictly positive penalty"),
])
def test_monotonic_preconditions(kw, msg):
    p, u = O.dense_fixture(6100, dim=3, steps=12, **kw)
    cfg = I.IsmConfig(subintervals=2, max_outer=2, eta=0.0, partition="uniform")
    sv = I.SolverSpec(kind="monotonic")
    for run in (lambda: O.ref_ism_run(p, u, cfg, sv), lambda: O.ism_run(p, u, cfg, sv, O.REFERENCE)):
        with pytest.raises(I.LogicError, match=msg):
            run()


def test_monotonic_rejects_matrix_states():
    w = problems.spins_preset(quick=True, subintervals=2, iterations=2, steps=16)
    w.config.workers = 1  # the reference's worker threads do not forward exceptions (runtime.cpp:29-49)
    sv = I.SolverSpec(kind="monotonic")
    for run in (lambda: O.ref_ism_run(w.problem, w.u0, w.config, sv),
                lambda: O.ism_run(w.problem, w.u0, w.config, sv, O.REFERENCE)):
        with pytest.raises(I.LogicError, match="column states"):
            run()


@pytest.mark.parametrize("dim,channels,alpha", [(3, 1, 3.0), (4, 2, 0.5)])
@pytest.mark.parametrize("parts", [1, 4])
def test_newton_gmres(dim, channels, alpha, parts):
    # The Hessian-vector products are central differences with h ~ hvp_scale (1e-5): they amplify
    # the last-bit differences between the two LU summation orders by ~1/h, and GMRES stops at a
    # relative residual of 1e-6 -- agreement is to 1e-7 of the control scale, not to rounding.
    p, u = O.dense_fixture(6200 + dim, dim=dim, steps=20, channels=channels, alpha=alpha)
    cfg = I.IsmConfig(subintervals=parts, max_outer=4, eta=0.0, partition="uniform")
    sv = I.SolverSpec(kind="newton", step_size=0.2)
    r, o = O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    compare_newton(r, o)
    assert _events(r) == _events(o)  # the same directions fell back to gradient steps


def compare_newton(r, o, ctl=1e-7, obj=1e-8):
    scale = max(1.0, float(np.max(np.abs(r.control))))
    assert np.max(np.abs(r.control - o.control)) <= ctl * scale
    assert len(r.record.iterations) == len(o.record.iterations)
    for a, b in zip(r.record.iterations, o.record.iterations):
        if np.isfinite(a.objective) or np.isfinite(b.objective):
            assert abs(a.objective - b.objective) <= obj
        if a.error is not None:
            assert abs(a.error - b.error) <= 1e-6 * max(1.0, abs(a.error))


def test_newton_on_the_condensate_split_variant():
    p, u = O.strang_fixture(3100)
    cfg = I.IsmConfig(subintervals=2, max_outer=2, eta=0.0, variant="split", partition="uniform")
    sv = I.SolverSpec(kind="newton", step_size=0.2, gmres_max_iter=12)
    compare_newton(O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv)[0])


# ---- a caller-defined potential (the virtual potential()/potential_derivative() plugin) ---------
@pytest.mark.parametrize("parts", [1, 2, 4])
@pytest.mark.parametrize("naive", [False, True])
def test_basis_potential_plugin(parts, naive):
    # the reference runs its own split-step path on a HamiltonianModel subclass defined in
    # oracle/ref_capi.cpp (BasisCondensate); the oracle evaluates the same separable form
    p, u = O.basis_fixture(6400)
    cfg = I.IsmConfig(subintervals=parts, max_outer=4, eta=0.0, variant="split", log_exact_objective=True,
                      partition="uniform")
    sv = I.SolverSpec(step_size=0.3, naive_nonlinear_adjoint=naive)
    compare(O.ref_ism_run(p, u, cfg, sv)[0], O.ism_run(p, u, cfg, sv)[0])


def test_basis_form_of_the_lattice_equals_the_lattice_kind():
    from paper_1603_01237_b200 import abi
    from paper_1603_01237_b200.models import BasisCondensateModel, CondensateModel
    p, u = O.basis_fixture(6401)
    lat = CondensateModel(32, -8.0, 8.0, abi.POT_LATTICE, [1.0, 5.0, 1.0], 1.5)
    bas = BasisCondensateModel.lattice(32, -8.0, 8.0, 1.0, 5.0, 1.0, 1.5)
    cfg = I.IsmConfig(subintervals=2, max_outer=3, eta=0.0, variant="split")
    sv = I.SolverSpec(step_size=0.3)
    a = O.ism_run(I.ControlProblem(lat, p.grid, p.initial, p.target, p.penalty), u, cfg, sv)[0]
    b = O.ism_run(I.ControlProblem(bas, p.grid, p.initial, p.target, p.penalty), u, cfg, sv)[0]
    compare(a, b, ctl_abs=1e-12, obj_abs=1e-12)


def test_stationary_state_matches_reference_ground_state():
    # problems.stationary_state (imaginary time + self-consistent diagonalisation) against the
    # reference's own ground_state (models.cpp:129-294): same discrete stationary state
    from paper_1603_01237_b200 import abi
    from paper_1603_01237_b200.models import CondensateModel
    for u in (0.0, 1.0):
        m = CondensateModel(50, -10.0, 10.0, abi.POT_TRAP, [6.0], 1.0)
        psi = problems.stationary_state(m, u)
        ref, energy, mu, residual, _ = O.ref_ground_state(50, -10.0, 10.0, 6.0, 1.0, u)
        assert residual < 1e-10
        assert np.max(np.abs(psi - ref)) < 1e-9

"""CPU oracle pins (no GPU): the reference's known-answer tests and property tests of the ISM
path, re-expressed against oracle/oracle.cpp.  These pin the checker the
device parity tests rely on.

KAT-2 (density-matrix J-coupling) and KAT-7 (efficiency CSV strings) are outside the hot
path (conjugation kind and CLI reporting); everything else on §8(c)'s list is here.
"""
import math

import numpy as np
import pytest

from paper_1603_01237_b200 import abi
from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import problems
from paper_1603_01237_b200.models import CondensateModel, DenseModel, TridiagonalModel
from tests import oracle_api as O


def scalar_problem(h, dt, steps=1, psi=1.0 + 0j):
    model = DenseModel(np.array([[h]], complex), np.zeros((1, 1, 1), complex))
    grid = I.TimeGrid(0.0, dt, steps)
    return I.ControlProblem(model, grid, np.array([psi]), np.array([psi]), np.zeros(steps))


# ---- KAT-1: scalar rational step (propagation_test.cpp:31-42) ------------------------------
def test_kat1_scalar_cayley_step():
    omega, dt = 1.37, 0.05
    psi = 0.6 - 0.8j
    p = scalar_problem(omega, dt)
    out = O.step(p, [0.0], dt, np.array([psi]), arith=O.REFERENCE)
    expect = psi * complex(1.0, -0.5 * dt * omega) / complex(1.0, 0.5 * dt * omega)
    assert abs(out[0] - expect) < 1e-15


# ---- KAT-3: trap potential two-branch formula (models_test.cpp:153-170) --------------------
def test_kat3_trap_potential():
    m = CondensateModel(24, -8.0, 8.0, abi.POT_TRAP, [6.0], 1.0)
    v = m.potential([1.0])
    assert v[12] == pytest.approx(36.0 / 16.0, rel=1e-12)
    assert v[0] == pytest.approx(12.5, rel=1e-14)


# ---- KAT-4: harmonic limit of the stationary solver (models_test.cpp:182-190) --------------
def test_kat4_harmonic_ground_state_energy():
    m = CondensateModel(64, -10.0, 10.0, abi.POT_TRAP, [10.0], 0.0)
    psi = problems.stationary_state(m, 0.0)
    hat = np.fft.fft(psi, norm="ortho")
    v = m.potential([0.0])
    energy = m.dx * (np.sum(m.kinetic * np.abs(hat) ** 2) + np.sum(v * np.abs(psi) ** 2))
    assert energy == pytest.approx(0.5, rel=1e-8)
    assert abs(math.sqrt(m.dx) * np.linalg.norm(psi) - 1.0) < 1e-12


# ---- KAT-6: penalty hand sum (controls_test.cpp:79-95) -------------------------------------
def test_kat6_penalty_hand_sum():
    p = scalar_problem(0.0, 0.25, steps=4)
    p.penalty = np.array([1.0, 0.5, 7.0, 2.0])
    u = np.array([[1.0, 2.0, 0.0, -2.0]])
    # tracking payoff is 0 (H = 0 keeps psi = target), so the value is -penalty
    val, _ = O.objective_gradient(p, u, "tracking", arith=O.REFERENCE)
    assert val[0] == pytest.approx(-1.375, rel=1e-15)


# ---- DFT vs a naive sum (linalg_test.cpp:61-72) --------------------------------------------
@pytest.mark.parametrize("n", [1, 8, 50, 64, 1024])
def test_dft_matches_naive_sum(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    k = np.arange(n)
    naive = np.exp(-2j * np.pi * np.outer(k, k) / n) @ x / math.sqrt(n)
    assert np.max(np.abs(O.dft(x) - naive)) < 1e-12
    assert np.max(np.abs(O.dft(O.dft(x), inverse=True) - x)) < 1e-12


# ---- norm conservation (acceptance criterion 5) --------------------------------------------
def test_norm_drift_per_cayley_step():
    w = problems.rotor21(subintervals=1, iterations=1, tridiagonal=True)
    p = I.ControlProblem(w.problem.model, I.TimeGrid(0.0, 1e-3, 400), w.problem.initial,
                         w.problem.target, np.zeros(400))
    u = np.random.default_rng(3).uniform(-0.2, 0.2, (1, 400))
    traj = O.propagate(p, u, arith=O.REFERENCE)[0]
    norms = np.linalg.norm(traj, axis=1)
    assert np.max(np.abs(np.diff(norms))) <= 1e-13


def test_split_step_norm_drift():
    w = problems.condensate_preset()
    fin = O.propagate_final(w.problem, w.u0)[0]
    dx = w.problem.model.dx
    n0 = math.sqrt(dx) * np.linalg.norm(w.problem.initial)
    assert abs(math.sqrt(dx) * np.linalg.norm(fin) - n0) <= 1e-10


# ---- Theorems 1 and 2 over the identity fixtures (acceptance criteria 1-2) ----------------
@pytest.mark.parametrize("index", [i for i in range(50) if i % 3 != 0][:20])
def test_theorem_identities(index):
    dim, channels, quad = 2 + index % 7, 1 + index % 2, index % 5 == 0
    parts = [1, 2, 4, 8][index % 4]
    p, u = O.dense_fixture(9000 + index, dim=dim, steps=64, channels=channels, quadratic=quad,
                           random_penalty=True)
    j, _ = O.objective_gradient(p, u, "tracking", arith=O.REFERENCE)
    fm, gm = O.verify_decomposition(p, u, parts, arith=O.REFERENCE)
    assert fm <= 1e-11 * (1.0 + abs(j[0]))
    assert gm <= 1e-10


# ---- exact gradients vs central differences (acceptance criterion 4) ----------------------
def _fd_ratio(p, u, form, entries):
    _, g = O.objective_gradient(p, u, form, arith=O.REFERENCE)
    h = 1e-6
    worst = 0.0
    for (c, j) in entries:
        up, um = u.copy(), u.copy()
        up[c, j] += h
        um[c, j] -= h
        fp, _ = O.objective_gradient(p, up, form, arith=O.REFERENCE)
        fm, _ = O.objective_gradient(p, um, form, arith=O.REFERENCE)
        fd = (fp[0] - fm[0]) / (2 * h)
        allowed = max(1e-10, 1e-6 * max(abs(fd), abs(g[0][c, j])))
        worst = max(worst, abs(fd - g[0][c, j]) / allowed)
    return worst


def test_gradient_matches_finite_differences_dense():
    p, u = O.dense_fixture(77, dim=5, steps=24, channels=2, quadratic=True, random_penalty=True)
    ents = [(c, j) for c in range(2) for j in range(0, 24, 5)]
    assert _fd_ratio(p, u, "tracking", ents) <= 1.0
    assert _fd_ratio(p, u, "overlap", ents) <= 1.0


def test_gradient_matches_finite_differences_split_step():
    p, u = O.strang_fixture(31)
    assert _fd_ratio(p, u, "overlap", [(0, j) for j in range(12)]) <= 1.0


# ---- adjointness of the one-step maps (propagation_test.cpp:142-162) ----------------------
def test_adjoint_step_is_exact_transpose():
    p, u = O.dense_fixture(5, dim=6, steps=4, channels=1)
    rng = np.random.default_rng(0)
    a = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    b = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    dt = p.grid.dt
    Ma = O.step(p, u[:, 0], dt, a, arith=O.REFERENCE)
    Mhb = O.step(p, u[:, 0], dt, b, adjoint=True, arith=O.REFERENCE)
    assert abs(np.vdot(b, Ma) - np.vdot(Mhb, a)) < 1e-14


# ---- propagator assembly (acceptance criterion 6) -----------------------------------------
@pytest.mark.parametrize("i", range(0, 10, 2))
def test_assembly_apply_and_compose(i):
    p, u = O.dense_fixture(9500 + i, dim=4, steps=64)
    whole = O.assemble_propagator(p, u, arith=O.REFERENCE)[0]
    direct = O.propagate_final(p, u, arith=O.REFERENCE)[0]
    assert np.linalg.norm(whole @ p.initial - direct) <= 1e-11
    chained = np.eye(4, dtype=complex)
    for n in range(4):
        sub = I.ControlProblem(p.model, I.TimeGrid(p.grid.node(16 * n), p.grid.dt, 16), p.initial,
                               p.target, p.penalty[16 * n:16 * n + 16])
        chained = O.assemble_propagator(sub, u[:, 16 * n:16 * n + 16], arith=O.REFERENCE)[0] @ chained
    assert np.max(np.abs(chained - whole)) <= 1e-10


# ---- run_ism properties (ism_test.cpp) -----------------------------------------------------
def test_single_interval_run_is_one_gradient_step():
    p, u = O.dense_fixture(2400)
    cfg = I.IsmConfig(subintervals=1, max_outer=1, eta=0.0)
    run = O.ism_run(p, u, cfg, I.SolverSpec(step_size=0.4), O.REFERENCE)[0]
    j0, g = O.objective_gradient(p, u, "tracking", arith=O.REFERENCE)
    assert np.array_equal(run.control, u + 0.4 * g[0])  # bitwise, ism_test.cpp:155-184
    its = run.record.iterations
    assert len(its) == 2 and its[0].error is None and its[1].error is not None
    assert its[0].objective == j0[0]
    assert its[0].task_values == [its[0].objective]
    j1, _ = O.objective_gradient(p, run.control, "tracking", arith=O.REFERENCE)
    assert its[1].objective == j1[0]


def test_subinterval_invariance_and_worker_determinism():
    p, u = O.dense_fixture(2600, random_penalty=True)
    sv = I.SolverSpec(step_size=0.5)
    base = O.ism_run(p, u, I.IsmConfig(subintervals=1, max_outer=10, eta=0.0), sv, O.REFERENCE)[0]
    for parts in (2, 4, 8):
        run = O.ism_run(p, u, I.IsmConfig(subintervals=parts, max_outer=10, eta=0.0), sv, O.REFERENCE)[0]
        assert np.max(np.abs(run.control - base.control)) <= 1e-10
    cfg = I.IsmConfig(subintervals=4, max_outer=10, eta=0.0)
    serial = O.ism_run(p, u, cfg, sv, O.REFERENCE, threads=1)[0]
    pooled = O.ism_run(p, u, cfg, sv, O.REFERENCE, threads=4)[0]
    assert np.array_equal(serial.control, pooled.control)
    for a, b in zip(serial.record.iterations, pooled.record.iterations):
        assert a.objective == b.objective and a.task_values == b.task_values


def test_nonuniform_partition_keeps_invariance():
    # balanced parts (K mod L != 0) keep Theorem 2 -- K = 64 into 7 and 12 parts
    p, u = O.dense_fixture(2601, random_penalty=True, steps=64)
    sv = I.SolverSpec(step_size=0.5)
    base = O.ism_run(p, u, I.IsmConfig(subintervals=1, max_outer=5, eta=0.0), sv, O.REFERENCE)[0]
    for parts in (7, 12):
        run = O.ism_run(p, u, I.IsmConfig(subintervals=parts, max_outer=5, eta=0.0), sv, O.REFERENCE)[0]
        assert np.max(np.abs(run.control - base.control)) <= 1e-10
    with pytest.raises(I.QocRuntimeError):
        O.ism_run(p, u, I.IsmConfig(subintervals=7, max_outer=1, partition="uniform"), sv, O.REFERENCE)


def test_direct_and_assembled_plans_agree():
    p, u = O.dense_fixture(2700, random_penalty=True)
    sv = I.SolverSpec(step_size=0.5)
    a = O.ism_run(p, u, I.IsmConfig(subintervals=4, max_outer=5, eta=0.0, plan="assembled"), sv)[0]
    d = O.ism_run(p, u, I.IsmConfig(subintervals=4, max_outer=5, eta=0.0, plan="direct"), sv)[0]
    assert np.max(np.abs(a.control - d.control)) < 1e-11


def test_eta_stop_and_record_shape():
    p, u = O.dense_fixture(2800)
    run = O.ism_run(p, u, I.IsmConfig(subintervals=2, max_outer=50, eta=1e9), I.SolverSpec(step_size=0.1))[0]
    assert len(run.record.iterations) == 2  # stops after the first iteration once error <= eta


def test_input_rejection():
    p, u = O.dense_fixture(2900)
    sv = I.SolverSpec(step_size=0.1)
    for bad in (I.IsmConfig(subintervals=0), I.IsmConfig(workers=0), I.IsmConfig(max_outer=-1),
                I.IsmConfig(eta=-1.0)):
        with pytest.raises(I.InvalidArgument):
            O.ism_run(p, u, bad, sv)
    with pytest.raises(I.LogicError):
        O.ism_run(p, u, I.IsmConfig(max_outer=1), I.SolverSpec(kind="monotonic"), O.REFERENCE)  # two channels


def test_split_variant_one_iteration_matches_single_interval():
    # ism_test.cpp:283-309: zero penalty; split N=4, one iteration == N=1 to 1e-12, and a
    # do-nothing solver keeps the lagged boundary data exact
    p, u = O.strang_fixture(3000, alpha=0.0)
    sv = I.SolverSpec(step_size=0.3)
    one = O.ism_run(p, u, I.IsmConfig(subintervals=1, max_outer=1, eta=0.0, variant="split"), sv)[0]
    four = O.ism_run(p, u, I.IsmConfig(subintervals=4, max_outer=1, eta=0.0, variant="split"), sv)[0]
    assert np.max(np.abs(one.control - four.control)) < 1e-12
    still = O.ism_run(p, u, I.IsmConfig(subintervals=4, max_outer=3, eta=0.0, variant="split"),
                      I.SolverSpec(step_size=0.0))[0]
    truth, _ = O.objective_gradient(p, u, "overlap")
    for it in still.record.iterations:
        assert it.objective == pytest.approx(truth[0], rel=1e-11)


# ---- KAT-8: the pinned condensate run (acceptance_main.cpp:439-485) ------------------------
def test_kat8_condensate_ten_iterations():
    w = problems.condensate_preset(subintervals=4, iterations=10)
    v0, _ = O.objective_gradient(w.problem, w.u0, "overlap")
    run = O.ism_run(w.problem, w.u0, w.config, w.solver)[0]
    pay = [it.exact_objective for it in run.record.iterations if it.exact_objective is not None]
    assert len(pay) == 10
    prev = v0[0]
    for v in pay:
        assert v > prev
        prev = v
    assert pay[-1] >= -0.742728295 - 1e-6


# ---- structured solves agree with the reference's dense LU ---------------------------------
def test_tridiagonal_thomas_matches_dense_lu():
    w = problems.rotor21(subintervals=8, iterations=3, rho=100.0)
    p = I.ControlProblem(w.problem.model, I.TimeGrid(0.0, 1e-3, 800), w.problem.initial, w.problem.target,
                         np.zeros(800))
    u = w.u0[:, :800]
    a = O.propagate_final(p, u, O.STRUCTURED)
    b = O.propagate_final(p, u, O.REFERENCE)
    assert np.max(np.abs(a - b)) < 1e-13
    _, ga = O.objective_gradient(p, u, "tracking", arith=O.STRUCTURED)
    _, gb = O.objective_gradient(p, u, "tracking", arith=O.REFERENCE)
    assert np.max(np.abs(ga - gb)) < 1e-13


def test_bitflip_neumann_matches_dense_lu():
    w = problems.ising10(nspins=5, steps=40, T=0.3)
    u = w.u0
    a = O.propagate_final(w.problem, u, O.STRUCTURED)
    b = O.propagate_final(w.problem, u, O.REFERENCE)
    assert np.max(np.abs(a - b)) < 1e-13
    _, ga = O.objective_gradient(w.problem, u, "tracking", arith=O.STRUCTURED)
    _, gb = O.objective_gradient(w.problem, u, "tracking", arith=O.REFERENCE)
    assert np.max(np.abs(ga - gb)) < 1e-13


def test_tridiagonal_model_round_trips_dense():
    w = problems.rotor21(subintervals=1, iterations=1)
    dense = w.problem.model.to_dense()
    back = TridiagonalModel.from_dense(dense)
    assert np.array_equal(back.diag, w.problem.model.diag)
    assert np.array_equal(back.sub, w.problem.model.sub)

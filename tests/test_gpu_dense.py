"""Device parity, dense operators: libqoc_b200.so vs the CPU oracle on the reference's own
seeded fixtures (fixtures.hpp:66-112) and BASELINE config 1."""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import problems
from tests import oracle_api as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("quad", [False, True])
@pytest.mark.parametrize("dim", [2, 4, 7, 16, 21, 33, 48, 64])
def test_propagate_gradient_assemble(ctx, quad, dim):
    p, u = O.dense_fixture(100 + dim + 2 * quad, dim=dim, steps=16, quadratic=quad, random_penalty=True)
    fin = I.propagate_final(p, u, ctx)
    ref = O.propagate_final(p, u, O.REFERENCE)
    assert np.max(np.abs(fin - ref)) < 1e-13
    for form in ("overlap", "tracking"):
        v, g = I.objective_gradient(p, u, form, ctx=ctx)
        vr, gr = O.objective_gradient(p, u, form, arith=O.REFERENCE)
        assert abs(v[0] - vr[0]) < 1e-13
        assert np.max(np.abs(g - gr)) < 1e-13
    M = I.assemble_propagator(p, u, ctx)
    Mr = O.assemble_propagator(p, u, O.REFERENCE)
    assert np.max(np.abs(M - Mr)) < 1e-13


@pytest.mark.parametrize("parts", [1, 2, 4, 8, 5])
@pytest.mark.parametrize("plan", ["assembled", "direct"])
def test_run_ism_matches_oracle(ctx, parts, plan):
    p, u = O.dense_fixture(2600, random_penalty=True)
    cfg = I.IsmConfig(subintervals=parts, max_outer=5, eta=0.0, plan=plan)
    sv = I.SolverSpec(step_size=0.5)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    assert np.max(np.abs(g.control - r.control)) < 1e-12
    assert len(g.record.iterations) == len(r.record.iterations) == 6
    for a, b in zip(g.record.iterations, r.record.iterations):
        assert a.iteration == b.iteration
        assert abs(a.objective - b.objective) < 1e-12
        assert (a.error is None) == (b.error is None)
        if a.error is not None:
            assert abs(a.error - b.error) < 1e-11 * max(1.0, abs(b.error))
        assert np.max(np.abs(np.array(a.task_values) - np.array(b.task_values))) < 1e-12


def test_spin2_200_iterations(ctx):
    for rho in (0.1, 10.0):
        w = problems.spin2(rho=rho)
        g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
        r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0]
        assert rel(g.control, r.control) < 1e-9
        assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-10


@pytest.mark.parametrize("disable", ["", "nm"])
def test_batch_subset(ctx, disable, monkeypatch):
    # the Neumann/tensor-core path and (QOC_DISABLE=nm, read per launch) the Gauss-Jordan path
    monkeypatch.setenv("QOC_DISABLE", disable)
    monkeypatch.setenv("QOC_ENABLE", "fuse" if disable == "" else "")
    w = problems.batch4096(batch=8, iterations=3)
    gs = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
    rs = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
    for g, r in zip(gs, rs):
        assert rel(g.control, r.control) < 1e-11
        assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-11


@pytest.mark.slow
def test_batch4096_problem_sample_long_run(ctx):
    # BASELINE config 5 at full problem size (d = 16, K = 2000, L = 128), SURVEY §8(d) parity
    # plan: 64 fixed problem indices (8 blocks of 8 spread over the 4096 seeds), 200 iterations
    # at rho = 0.1/dt
    # at rho = 0.1/dt and at the literal rho = 0.1
    for fast in (True, False):
        for first in range(0, 4096, 512):
            w = problems.batch4096(batch=8, iterations=200, first=first)
            if fast:
                w.solver.step_size = w.rho_fast
            gs = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
            rs = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
            for g, r in zip(gs, rs):
                assert rel(g.control, r.control) < 1e-9
                assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-10


def test_batch_neumann_range_handoff(ctx):
    # config-5 kind (d = 16, one linear control): the Neumann-in-the-control assembly covers
    # |u| a ||Hc||_1 up to its staged term count; tasks past it (problem 1: every task; problem
    # 2: one subinterval; problem 3: far enough that a ||H(u)||_1 >= 1, the partial-pivoting
    # Gauss-Jordan path) are handed to the Gauss-Jordan kernel -- results match the oracle
    w = problems.batch4096(batch=4, iterations=4, subintervals=16)
    u0 = np.array(w.u0)
    u0[1] *= 100.0
    u0[2, 0, 500:625] *= 100.0
    u0[3] *= 1500.0
    w.solver.step_size = 0.5
    gs = I.run_ism_batch(w.problem, u0, w.config, w.solver, ctx)
    rs = O.ism_run(w.problem, u0, w.config, w.solver, O.REFERENCE)
    for g, r in zip(gs, rs):
        assert not r.record.aborted
        assert rel(g.control, r.control) < 1e-11
        assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-11
        for a, b in zip(g.record.iterations[1:], r.record.iterations[1:]):
            assert abs(a.error - b.error) < 1e-10 * max(1.0, abs(b.error))


def test_batch_all_problems_two_iterations(ctx):
    # SURVEY §8(d) / VERDICT r01: every one of the 4096 config-5 problems for 2 outer iterations
    # at both step sizes; the oracle runs the same batch on all host threads
    for fast in (False, True):
        w = problems.batch4096(iterations=2)
        if fast:
            w.solver.step_size = w.rho_fast
        gs = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
        rs = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
        du = max(rel(g.control, r.control) for g, r in zip(gs, rs))
        dobj = max(np.max(np.abs(g.record.objectives() - r.record.objectives())) for g, r in zip(gs, rs))
        derr = max(abs(a.error - b.error) / max(1.0, abs(b.error))
                   for g, r in zip(gs, rs) for a, b in zip(g.record.iterations[1:], r.record.iterations[1:]))
        assert du < 1e-9 and dobj < 1e-10 and derr < 1e-9, (fast, du, dobj, derr)


@pytest.mark.parametrize("dim", [48, 64])
@pytest.mark.parametrize("variant,plan", [("interpolated", "assembled"), ("interpolated", "direct"),
                                          ("split", "assembled")])
def test_run_ism_large_dense(ctx, dim, variant, plan):
    # DenseModel beyond the warp-resident sizes (CTA-per-task kernels, dense_big.cu); the
    # reference benchmarks a d = 64 Crank-Nicolson step (benchmarks.cpp:76)
    p, u = O.dense_fixture(2650 + dim, dim=dim, steps=12, channels=2, quadratic=True, random_penalty=True)
    cfg = I.IsmConfig(subintervals=3, max_outer=9, eta=0.0, variant=variant, plan=plan,
                      log_exact_objective=(variant == "split"))
    sv = I.SolverSpec(step_size=0.5)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    assert rel(g.control, r.control) < 1e-12
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-12
    for a, b in zip(g.record.iterations[1:], r.record.iterations[1:]):
        assert abs(a.error - b.error) < 1e-11 * max(1.0, abs(b.error))


def test_dense_above_64_rejected(ctx):
    p, u = O.dense_fixture(2690, dim=65, steps=4, channels=1)
    with pytest.raises(I.LogicError):
        I.run_ism(p, u, I.IsmConfig(subintervals=2, max_outer=1), I.SolverSpec(step_size=0.1), ctx)

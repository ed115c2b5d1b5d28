"""The one-pass iteration of the Neumann path (dense d = 16, one control; driver.cu `onepass`).

It evaluates the residual of iteration k and the entry value + update of iteration k + 1 in one
streaming pass over the propagator cache and applies that update at the start of k + 1 -- the
same arithmetic as the gradient -> assembly -> residual order, reordered.  So the two orders
must agree BIT FOR BIT (QOC_DISABLE=onepass selects the two-pass order), and both must match
the oracle through the stop and abort paths the reorder moves across: the eta stop, the
non-finite-control abort (ism.cpp:527-539) and single-subinterval runs.
"""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import problems
from tests import oracle_api as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def workload(batch, iterations, subintervals=128, K=2000):
    """BASELINE config 5's problems (d = 16, one control); the Neumann path needs <= 32 steps
    per subinterval, so K = 2000 takes >= 63 subintervals and a single-subinterval run K <= 32."""
    w = problems.batch4096(batch=batch, iterations=iterations, subintervals=subintervals)
    if K != 2000:
        h0, hc, psi_i, psi_t, u0 = problems.batch_problems(batch, 16, 1000, 100000, K)
        grid = I.TimeGrid.over(0.0, 10.0 * K / 2000, K)
        w.problem = I.ControlProblem(type(w.problem.model)(h0, hc[:, None]), grid, psi_i, psi_t, np.zeros(K))
        w.u0 = u0
    return w


def both_orders(ctx, monkeypatch, w, u0=None):
    u0 = w.u0 if u0 is None else u0
    one = I.run_ism_batch(w.problem, u0, w.config, w.solver, ctx)
    monkeypatch.setenv("QOC_DISABLE", "onepass")
    two = I.run_ism_batch(w.problem, u0, w.config, w.solver, ctx)
    monkeypatch.delenv("QOC_DISABLE")
    return one, two


def same_bits(a, b):
    assert np.array_equal(a.control, b.control, equal_nan=True)
    assert np.array_equal(a.record.objectives(), b.record.objectives(), equal_nan=True)
    ea = [it.error for it in a.record.iterations]
    eb = [it.error for it in b.record.iterations]
    assert ea == eb
    ta = np.array([it.task_values for it in a.record.iterations])
    tb = np.array([it.task_values for it in b.record.iterations])
    assert np.array_equal(ta, tb, equal_nan=True)
    assert a.record.aborted == b.record.aborted and a.record.abort_reason == b.record.abort_reason


@pytest.mark.parametrize("parts,iters,K", [(128, 12, 2000), (100, 3, 2000), (1, 9, 24), (3, 10, 32)])
def test_onepass_bitwise_equals_two_pass(ctx, monkeypatch, parts, iters, K):
    w = workload(5, iters, parts, K)
    w.solver.step_size = w.rho_fast
    one, two = both_orders(ctx, monkeypatch, w)
    for a, b in zip(one, two):
        same_bits(a, b)
    rs = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
    for g, r in zip(one, rs):
        assert rel(g.control, r.control) < 1e-11
        assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-11


def test_onepass_eta_stop_mid_run(ctx, monkeypatch):
    # an eta between the members' residuals: they stop at different iterations
    w = workload(4, 12)
    probe = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
    errs = sorted(r.record.iterations[4].error for r in probe)
    w.config.eta = 0.5 * (errs[1] + errs[2])
    one, two = both_orders(ctx, monkeypatch, w)
    rs = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
    lens = set()
    for a, b, r in zip(one, two, rs):
        same_bits(a, b)
        assert len(a.record.iterations) == len(r.record.iterations)
        lens.add(len(a.record.iterations))
        assert rel(a.control, r.control) < 1e-11
    assert len(lens) > 1  # the members really stopped at different iterations


def test_onepass_abort_mid_run(ctx, monkeypatch):
    # a penalty with an absurd step multiplies the controls by ~ -1e20 per iteration
    # (g_j = -alpha dt u_j + ...), so they overflow mid-run (the Neumann range check hands the
    # tasks to Gauss-Jordan on the way): the run aborts with the reference's reason and returns
    # the abort iteration's control
    w = workload(2, 24, 64)
    w.problem.penalty = np.full(w.problem.grid.steps, 1.0)
    w.solver.step_size = 1e20 / (w.problem.grid.dt * w.problem.grid.steps / 64)
    one, two = both_orders(ctx, monkeypatch, w)
    rs = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
    for a, b, r in zip(one, two, rs):
        same_bits(a, b)
        assert r.record.aborted and a.record.aborted
        assert a.record.abort_reason == r.record.abort_reason
        assert len(a.record.iterations) == len(r.record.iterations)
        assert 3 < len(a.record.iterations) < 25
        assert np.array_equal(np.isfinite(a.control), np.isfinite(r.control))

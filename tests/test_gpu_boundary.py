"""Device parity at the edges of the C-ABI contract (ADVICE r01 / VERDICT r01 "silent wrong
results at the boundary"):

* DenseModel / tridiagonal models with C = 5 and 6 control channels (models.cpp:57-75 takes any
  C) through run_ism, objective_gradient and the propagator-cache engine; C above the device
  bound is rejected with std::logic_error, never truncated;
* the abort path returns the control of the abort iteration (ism.cpp:527-539, 611);
* GradientOptions::naive_nonlinear_adjoint reaches the split-step task and node sweeps
  (ism.cpp:373,437,446,543);
* run_inner with inner_iterations 0 (entry value only) and 2 (optimizers.cpp:261-285).
"""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200.models import DenseModel, TridiagonalModel
from tests import oracle_api as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def many_channel_fixture(seed, dim, channels, quadratic=False, steps=24, tridiagonal=False):
    rng = np.random.default_rng(seed)

    def herm(scale=1.0):
        g = rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))
        h = (g + g.conj().T) / 2 * scale
        if tridiagonal:
            band = np.abs(np.subtract.outer(np.arange(dim), np.arange(dim))) > 1
            h[band] = 0
        return h

    h0 = herm()
    lin = np.stack([herm(0.5) for _ in range(channels)])
    quad = np.stack([herm(0.2) for _ in range(channels)]) if quadratic else None
    model = DenseModel(h0, lin, quad)
    if tridiagonal:
        model = TridiagonalModel.from_dense(model)
    v = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    w = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    grid = I.TimeGrid.over(0.0, 1.0, steps)
    p = I.ControlProblem(model, grid, v / np.linalg.norm(v), w / np.linalg.norm(w), np.full(steps, 0.05))
    u = 0.3 * rng.standard_normal((channels, steps))
    return p, u


@pytest.mark.parametrize("channels", [5, 6])
@pytest.mark.parametrize("quad", [False, True])
def test_dense_many_channels(ctx, channels, quad):
    p, u = many_channel_fixture(40 + channels, 6, channels, quad)
    for form in ("overlap", "tracking"):
        v, g = I.objective_gradient(p, u, form, ctx=ctx)
        vr, gr = O.objective_gradient(p, u, form, arith=O.REFERENCE)
        assert abs(v[0] - vr[0]) < 1e-13
        assert np.max(np.abs(g - gr)) < 1e-13
    for parts in (1, 4, 5):
        cfg = I.IsmConfig(subintervals=parts, max_outer=10, eta=0.0)  # >= 8: graph replay
        sv = I.SolverSpec(step_size=0.5)
        gr_ = I.run_ism(p, u, cfg, sv, ctx)
        r = O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
        assert rel(gr_.control, r.control) < 1e-12
        # every channel moved (none silently frozen at its initial value)
        assert np.all(np.max(np.abs(gr_.control - u), axis=1) > 0)
        assert np.max(np.abs(gr_.record.objectives() - r.record.objectives())) < 1e-12
        for a, b in zip(gr_.record.iterations, r.record.iterations):
            if b.error is not None:
                assert abs(a.error - b.error) < 1e-11 * max(1.0, abs(b.error))


@pytest.mark.parametrize("channels", [5, 6])
def test_tridiagonal_many_channels(ctx, channels):
    p, u = many_channel_fixture(60 + channels, 9, channels, tridiagonal=True)
    v, g = I.objective_gradient(p, u, "tracking", ctx=ctx)
    vr, gr = O.objective_gradient(p, u, "tracking", arith=O.REFERENCE)
    assert np.max(np.abs(g - gr)) < 1e-13
    cfg = I.IsmConfig(subintervals=4, max_outer=9, eta=0.0)
    sv = I.SolverSpec(step_size=0.5)
    gr_ = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    assert rel(gr_.control, r.control) < 1e-12
    assert np.all(np.max(np.abs(gr_.control - u), axis=1) > 0)


def test_too_many_channels_rejected(ctx):
    p, u = many_channel_fixture(7, 4, 9)
    with pytest.raises(I.LogicError):
        I.run_ism(p, u, I.IsmConfig(subintervals=2, max_outer=1), I.SolverSpec(step_size=0.1), ctx)
    with pytest.raises(I.LogicError):
        I.objective_gradient(p, u, ctx=ctx)


@pytest.mark.parametrize("parts", [1, 4])
def test_abort_returns_abort_iteration_control(ctx, parts):
    p, u = O.dense_fixture(2700, random_penalty=True)
    cfg = I.IsmConfig(subintervals=parts, max_outer=40, eta=0.0)
    sv = I.SolverSpec(step_size=1e300)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv)[0]
    assert r.record.aborted and g.record.aborted
    assert g.record.abort_reason == r.record.abort_reason
    assert len(g.record.iterations) == len(r.record.iterations)
    # same non-finite pattern and the same finite values (ism.cpp:611 returns concat(u_parts))
    assert np.array_equal(np.isfinite(g.control), np.isfinite(r.control))
    fin = np.isfinite(r.control)
    assert np.allclose(g.control[fin], r.control[fin], rtol=1e-12, atol=0)


def test_batch_abort_freezes_only_that_problem(ctx):
    # one problem of a batch aborts in the bootstrap (a non-finite first-guess sample makes its
    # boundary states non-finite, ism.cpp:385-391); its control must come back untouched while
    # the other member keeps iterating
    from paper_1603_01237_b200 import problems
    w = problems.batch4096(batch=2, iterations=10, subintervals=4)
    u0 = np.array(w.u0)
    u0[1, 0, 5] = np.inf
    w.solver.step_size = 20.0
    gs = I.run_ism_batch(w.problem, u0, w.config, w.solver, ctx)
    rs = O.ism_run(w.problem, u0, w.config, w.solver, O.REFERENCE)
    assert rs[1].record.aborted and gs[1].record.aborted and not gs[0].record.aborted
    assert gs[1].record.abort_reason == rs[1].record.abort_reason
    assert len(gs[1].record.iterations) == len(rs[1].record.iterations) == 1
    assert np.array_equal(gs[1].control, u0[1]) and np.array_equal(rs[1].control, u0[1])
    assert rel(gs[0].control, rs[0].control) < 1e-11


@pytest.mark.parametrize("plan", ["assembled", "direct"])
def test_naive_adjoint_reaches_the_run(ctx, plan):
    p, u = O.strang_fixture(3100, steps=16)
    cfg = I.IsmConfig(subintervals=4, max_outer=4, eta=0.0, variant="split", plan=plan, log_exact_objective=True)
    sv = I.SolverSpec(step_size=0.3, naive_nonlinear_adjoint=True)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv)[0]
    assert rel(g.control, r.control) < 1e-12
    exact = I.SolverSpec(step_size=0.3)
    rx = O.ism_run(p, u, cfg, exact)[0]
    assert rel(rx.control, r.control) > 1e-8  # the flag changes the answer, and the device follows it


@pytest.mark.parametrize("inner", [0, 2])
@pytest.mark.parametrize("kind", ["dense", "rotor", "strang"])
def test_inner_iterations(ctx, inner, kind):
    if kind == "dense":
        p, u = O.dense_fixture(2611, random_penalty=True)
        cfg = I.IsmConfig(subintervals=4, max_outer=9, eta=0.0)
        arith = O.REFERENCE
    elif kind == "rotor":
        from paper_1603_01237_b200 import problems
        w = problems.rotor21(subintervals=8, iterations=9, rho=100.0)
        p, u, cfg = w.problem, w.u0, w.config
        p.grid = I.TimeGrid.over(0.0, 0.4, 400)
        u = np.asarray(u)[:, :400]
        p.penalty = None
        arith = O.STRUCTURED
    else:
        p, u = O.strang_fixture(3200, steps=16)
        cfg = I.IsmConfig(subintervals=4, max_outer=3, eta=0.0, variant="split")
        arith = O.STRUCTURED
    sv = I.SolverSpec(step_size=0.4 if kind != "rotor" else 100.0, inner_iterations=inner)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv, arith)[0]
    assert rel(g.control, r.control) < 1e-11
    if inner == 0:
        assert np.array_equal(g.control, np.asarray(u, dtype=np.float64).reshape(g.control.shape))
    ok = np.isfinite(r.record.objectives())
    assert np.max(np.abs(g.record.objectives()[ok] - r.record.objectives()[ok])) < 1e-11
    for a, b in zip(g.record.iterations, r.record.iterations):
        assert np.max(np.abs(np.array(a.task_values) - np.array(b.task_values))) < 1e-11

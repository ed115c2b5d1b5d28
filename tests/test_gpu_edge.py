"""Device edge cases of run_ism (ism.cpp:213-231,385-391,527-539,589-591): input rejection,
the eta stop, one-step subintervals, ragged partitions, and the numerical abort path, each
compared with the CPU oracle."""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from tests import oracle_api as O

pytestmark = pytest.mark.gpu


def test_input_rejection_matches_reference(ctx):
    p, u = O.dense_fixture(2900)
    sv = I.SolverSpec(step_size=0.1)
    for bad in (I.IsmConfig(subintervals=0), I.IsmConfig(workers=0), I.IsmConfig(max_outer=-1),
                I.IsmConfig(eta=-1.0)):
        with pytest.raises(I.InvalidArgument):
            I.run_ism(p, u, bad, sv, ctx)
    with pytest.raises(I.LogicError):
        I.run_ism(p, u, I.IsmConfig(max_outer=1), I.SolverSpec(kind="monotonic"), ctx)  # two channels
    with pytest.raises(I.QocRuntimeError):  # Decomposition::uniform with K % L != 0
        I.run_ism(p, u, I.IsmConfig(subintervals=5, max_outer=1, partition="uniform"), sv, ctx)
    with pytest.raises(I.QocRuntimeError):  # more parts than steps
        I.run_ism(p, u, I.IsmConfig(subintervals=p.grid.steps + 1, max_outer=1), sv, ctx)


def test_eta_stop(ctx):
    p, u = O.dense_fixture(2800)
    cfg = I.IsmConfig(subintervals=2, max_outer=50, eta=1e9)
    g = I.run_ism(p, u, cfg, I.SolverSpec(step_size=0.1), ctx)
    r = O.ism_run(p, u, cfg, I.SolverSpec(step_size=0.1))[0]
    assert len(g.record.iterations) == len(r.record.iterations) == 2
    assert np.max(np.abs(g.control - r.control)) < 1e-13


@pytest.mark.parametrize("parts", [16, 11])  # one-step tasks (L = K) and a ragged partition
def test_extreme_partitions(ctx, parts):
    p, u = O.dense_fixture(2601, steps=16, random_penalty=True)
    cfg = I.IsmConfig(subintervals=parts, max_outer=12, eta=0.0)  # >= 8 iterations: graph replay
    sv = I.SolverSpec(step_size=0.5)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv, O.REFERENCE)[0]
    assert np.max(np.abs(g.control - r.control)) < 1e-12
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-12


def test_abort_on_non_finite_controls(ctx):
    # an absurd step drives the controls to inf/nan: the run stops with the reference's reason
    p, u = O.dense_fixture(2700, random_penalty=True)
    cfg = I.IsmConfig(subintervals=4, max_outer=40, eta=0.0)
    sv = I.SolverSpec(step_size=1e300)
    g = I.run_ism(p, u, cfg, sv, ctx)
    r = O.ism_run(p, u, cfg, sv)[0]
    assert r.record.aborted and g.record.aborted
    assert g.record.abort_reason == r.record.abort_reason
    assert len(g.record.iterations) == len(r.record.iterations)


def test_batch_members_stop_independently(ctx):
    # two problems of a batch: the per-problem stop/abort state lives on the device
    from paper_1603_01237_b200 import problems
    w = problems.batch4096(batch=3, iterations=12, subintervals=8)
    gs = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
    rs = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
    for g, r in zip(gs, rs):
        assert np.max(np.abs(g.control - r.control)) / np.max(np.abs(r.control)) < 1e-11
        assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-11


@pytest.mark.parametrize("kind", ["batch", "rotor", "bitflip", "strang", "density", "gpe256", "newton", "monotonic"])
def test_run_to_run_bitwise_determinism(ctx, kind):
    # fixed-order reductions everywhere (no atomics on the data path): two runs of the same
    # problem give bit-identical controls and records (acceptance_main.cpp:143-157 asks the same
    # of the reference across worker counts)
    from paper_1603_01237_b200 import problems
    if kind == "batch":
        w = problems.batch4096(batch=16, iterations=9)
        w.solver.step_size = w.rho_fast
    elif kind == "rotor":
        w = problems.rotor21(subintervals=32, iterations=9, rho=100.0)
    elif kind == "bitflip":
        w = problems.ising10(nspins=7, steps=64, T=0.5, iterations=4, subintervals=8, rho=2.0)
    elif kind == "density":  # assembled plan, tensor-core products, kept inverses
        w = problems.spins_preset(quick=False, subintervals=8, iterations=4, steps=256)
    elif kind == "gpe256":  # merged kinetic half steps, compile-time FFT stages
        w = problems.gpe1024(subintervals=8, iterations=4, rho=5.0, points=256, steps=400, T=0.2)
    elif kind in ("newton", "monotonic"):
        p, u = O.dense_fixture(7003, dim=3, steps=24, channels=1, quadratic=True, alpha=1.0)
        cfg = I.IsmConfig(subintervals=4, max_outer=4, eta=0.0)
        w = type("W", (), {"problem": p, "u0": u, "config": cfg, "solver": I.SolverSpec(kind=kind, step_size=0.2)})
    else:
        p, u = O.strang_fixture(3300, steps=24)
        cfg = I.IsmConfig(subintervals=4, max_outer=9, eta=0.0, variant="split", log_exact_objective=True)
        w = type("W", (), {"problem": p, "u0": u, "config": cfg, "solver": I.SolverSpec(step_size=0.3)})
    a = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
    b = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
    for x, y in zip(a, b):
        assert np.array_equal(x.control, y.control)
        assert np.array_equal(x.record.objectives(), y.record.objectives(), equal_nan=True)
        for s, t in zip(x.record.iterations, y.record.iterations):
            assert np.array_equal(np.asarray(s.task_values), np.asarray(t.task_values), equal_nan=True)
            assert (s.error == t.error) or (s.error is None and t.error is None)


def test_checkpoint_stride_gives_identical_results(ctx):
    # CheckpointedTrajectory (propagation.cpp:202-234) only trades memory for recomputation: the
    # reference requires bit-identical results for any stride; the device keeps trajectories in
    # HBM/L2 and accepts the stride, and the oracle run with the same stride agrees
    p, u = O.strang_fixture(3000)
    base = I.IsmConfig(subintervals=4, max_outer=4, eta=0.0, variant="split", log_exact_objective=True)
    strided = I.IsmConfig(subintervals=4, max_outer=4, eta=0.0, variant="split", log_exact_objective=True,
                          checkpoint_stride=3)
    sv = I.SolverSpec(step_size=0.3, checkpoint_stride=3)
    a = I.run_ism(p, u, base, I.SolverSpec(step_size=0.3), ctx)
    b = I.run_ism(p, u, strided, sv, ctx)
    assert np.array_equal(a.control, b.control)
    r = O.ism_run(p, u, strided, sv)[0]
    assert np.max(np.abs(b.control - r.control)) < 1e-12


def test_run_artifacts_from_a_device_run(ctx, tmp_path):
    # `qoc run` artifacts (tools/main.cpp:178-200) written from a device run, and the `qoc bench`
    # efficiency.csv (main.cpp:339-372) over device runs at L = 1, 2, 4
    import json
    from paper_1603_01237_b200 import problems, wire
    w = problems.spin2(iterations=30, rho=10.0)
    run = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    wire.write_run_artifacts(tmp_path / "run", w.problem, run, {"preset": "spin2"})
    lines = (tmp_path / "run" / "iterations.jsonl").read_text().splitlines()
    assert len(lines) == 31 and json.loads(lines[5])["iteration"] == 5
    summary = json.loads((tmp_path / "run" / "summary.json").read_text())
    assert summary["result"]["iterations"] == 30 and summary["result"]["solver"] == "gradient"
    assert (tmp_path / "run" / "control.csv").read_text().startswith("t,")
    runs = []
    for L in (1, 2, 4):
        w.config.subintervals = L
        runs.append((L, I.run_ism(w.problem, w.u0, w.config, w.solver, ctx).record))
    csv = wire.bench_efficiency_csv(runs, [0.1, 0.01])
    rows = csv.splitlines()
    assert rows[0] == "eps,N,t_seconds,speedup,efficiency" and len(rows) == 7
    assert all(r.split(",")[0] in ("0.1", "0.01") for r in rows[1:])

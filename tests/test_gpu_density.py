"""Device parity, density-matrix conjugation kind (QOC_KIND_DENSITY): the
reference's `spins` preset (models.cpp:320-347 -- the paper's 5-spin benchmark)
with rho' = A rho A^dag steps (propagation.cpp:92-129) and the trace gradient of
objective.cpp:61-71, on the CTA-per-task kernels of dense_big.cu, vs the CPU oracle (itself pinned
to the reference's own cn_conjugation path, tests/test_reference_pinning.py)."""
import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import problems
from tests import oracle_api as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("quick", [True, False])
def test_propagate_gradient_assemble(ctx, quick):
    w = problems.spins_preset(quick=quick, steps=64)
    p, u = w.problem, w.u0
    fin = I.propagate_final(p, u, ctx)
    ref = O.propagate_final(p, u, O.REFERENCE)
    assert fin.shape == ref.shape == (1,) + (p.model.state_dim(),) * 2
    assert np.max(np.abs(fin - ref)) < 1e-12
    for form in ("overlap", "tracking"):
        v, g = I.objective_gradient(p, u, form, ctx=ctx)
        vr, gr = O.objective_gradient(p, u, form, arith=O.REFERENCE)
        assert abs(v[0] - vr[0]) < 1e-12 * max(1.0, abs(vr[0]))
        assert np.max(np.abs(g - gr)) < 1e-11 * max(1.0, np.max(np.abs(gr)))
    M = I.assemble_propagator(p, u, ctx)
    Mr = O.assemble_propagator(p, u, O.REFERENCE)
    assert np.max(np.abs(M - Mr)) < 1e-12


@pytest.mark.parametrize("parts", [1, 4, 8])
@pytest.mark.parametrize("variant", ["interpolated", "split"])
def test_spins_preset_run(ctx, parts, variant):
    # quick preset: 3 spins, 2^10 steps, rho = 1e4, 25 outer iterations (>= 8: graph replay)
    w = problems.spins_preset(quick=True, subintervals=parts)
    w.config.variant = variant
    w.config.log_exact_objective = variant == "split"
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0]
    assert len(g.record.iterations) == len(r.record.iterations) == 26
    assert rel(g.control - w.u0, r.control - w.u0) < 1e-9  # the update itself
    assert rel(g.control, r.control) < 1e-12
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-10
    for a, b in zip(g.record.iterations[1:], r.record.iterations[1:]):
        assert abs(a.error - b.error) < 1e-9 * max(1.0, abs(b.error))
        assert np.max(np.abs(np.asarray(a.task_values) - np.asarray(b.task_values))) < 1e-10


def test_five_spin_chain(ctx):
    # the paper's 5-spin chain (d = 32, 10 channels), shortened grid
    w = problems.spins_preset(quick=False, subintervals=8, iterations=6, steps=512)
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0]
    assert rel(g.control - w.u0, r.control - w.u0) < 1e-9
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-10


@pytest.mark.parametrize("variant", ["interpolated", "split"])
def test_assembled_and_direct_plans(ctx, variant):
    # the assembled plan chains the tasks' dm x dm products as prop * rho * prop^dag
    # (apply_propagator, propagation.cpp:251-261); the direct plan sweeps the nodes serially.
    # Both match the oracle's plan of the same name, and each other in the interpolated variant
    # (ism_test.cpp:248-265).
    w = problems.spins_preset(quick=True, subintervals=8, iterations=5)
    w.config.variant = variant
    runs = {}
    for plan in ("assembled", "direct"):
        w.config.plan = plan
        g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
        r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)[0]
        assert rel(g.control - w.u0, r.control - w.u0) < 1e-9
        assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-10
        assert g.record.plan == plan
        runs[plan] = g
    if variant == "interpolated":  # the split variant's assembled plan is the LAGGED refresh: a different iteration
        assert rel(runs["assembled"].control - w.u0, runs["direct"].control - w.u0) < 1e-9
        assert np.max(np.abs(runs["assembled"].record.objectives() - runs["direct"].record.objectives())) < 1e-11


def test_five_spin_tensor_core_products_match_cuda_cores(ctx):
    # QOC_DISABLE=densmma is read once per process, so the A/B runs in a subprocess: the fp64
    # tensor-core (DMMA) products and the CUDA-core products give the same run to rounding
    import json, os, subprocess, sys
    code = ("import json,sys; sys.path.insert(0,'.');"
            "from paper_1603_01237_b200 import ism as I, problems;"
            "w=problems.spins_preset(quick=False, subintervals=8, iterations=4, steps=256);"
            "g=I.run_ism(w.problem,w.u0,w.config,w.solver);"
            "print(json.dumps({'u':g.control.tolist(),'obj':g.record.objectives().tolist()}))")
    root = __import__("pathlib").Path(__file__).resolve().parents[1]
    outs = []
    for env in ({}, {"QOC_DISABLE": "densmma"}):
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root, timeout=600,
                           env={**os.environ, **env})
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    a, b = (np.array(o["u"]) for o in outs)
    w = problems.spins_preset(quick=False, subintervals=8, iterations=4, steps=256)
    assert rel(a - w.u0, b - w.u0) < 1e-9
    assert np.nanmax(np.abs(np.array(outs[0]["obj"]) - np.array(outs[1]["obj"]))) < 1e-11

"""Device parity of the blocked boundary refresh (bit-flip kind, SURVEY §8(e) option A): the G
block products P_g (d column sweeps per block), their chain into the block-boundary nodes and
the interior node sweeps, against the CPU oracle's direct plan.  The reference's own statement
of the equivalence is its direct-vs-assembled test (ism_test.cpp:248-265, < 1e-11); blocks = L
is the reference's per-subinterval assembled chain (ism.cpp:298-312).

On one GPU the G blocks are G emulated ranks in one launch sequence (the multi-rank exchange is
one in-place all-gather of the same slabs); the NCCL path itself runs here as a one-rank
communicator (tests/test_partition_gloo.py covers the host-side exchange at world size 2)."""
import numpy as np
import pytest

from paper_1603_01237_b200 import _native
from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import problems
from tests import oracle_api as O
from tests.test_gpu_bitflip import FIXTURES, compare_run, rel

pytestmark = pytest.mark.gpu


def _exact(run):
    return np.array([np.nan if it.exact_objective is None else it.exact_objective for it in run.record.iterations])


@pytest.mark.parametrize("nspins,parts,blocks", [(6, 7, 1), (6, 7, 2), (6, 7, 3), (6, 7, 7), (10, 8, 4),
                                                 (9, 12, 5)])
def test_blocked_matches_direct_oracle(ctx, nspins, parts, blocks):
    w = problems.ising10(nspins=nspins, steps=64, T=0.5, iterations=4, subintervals=parts, rho=2.0)
    w.config.plan, w.config.blocks = "assembled", blocks
    w.config.log_exact_objective = True
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    w.config.plan, w.config.blocks = "direct", 0
    r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0]
    assert rel(g.control, r.control) < 1e-11
    assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-11
    ex, exr = _exact(g), _exact(r)
    assert np.all(np.isfinite(ex[1:])) and np.max(np.abs(ex[1:] - exr[1:])) < 1e-11
    for a, b in zip(g.record.iterations[1:], r.record.iterations[1:]):
        assert abs(a.error - b.error) < 1e-10 * max(1.0, abs(b.error))
        assert np.max(np.abs(np.asarray(a.task_values) - np.asarray(b.task_values))) < 1e-11


def test_blocked_matches_device_direct_plan(ctx):
    # same device, both plans: agreement to rounding (ism_test.cpp:248-265 bound)
    w = problems.ising10(nspins=8, steps=96, T=0.7, iterations=9, subintervals=12, rho=3.0)
    d = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    for blocks in (4, 12):
        w.config.plan, w.config.blocks = "assembled", blocks
        b = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
        assert rel(b.control, d.control) < 1e-11
        assert np.max(np.abs(b.record.objectives() - d.record.objectives())) < 1e-11


def test_blocked_rejects_bad_block_counts(ctx):
    w = problems.ising10(nspins=6, steps=32, T=0.3, iterations=1, subintervals=4)
    w.config.plan = "assembled"
    for blocks, exc in ((5, I.InvalidArgument), (-1, I.InvalidArgument)):
        w.config.blocks = blocks
        with pytest.raises(exc):
            I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)


def test_blocked_through_one_rank_nccl_communicator():
    # the exchange path (pack -> in-place ncclAllGather -> unpack) on a one-rank communicator
    c = _native.Context()
    c.init_comm(0, 1, _native.comm_unique_id())
    try:
        w = problems.ising10(nspins=7, steps=48, T=0.4, iterations=3, subintervals=6, rho=2.0)
        w.config.plan, w.config.blocks = "assembled", 3
        g = I.run_ism(w.problem, w.u0, w.config, w.solver, c)
        w.config.plan, w.config.blocks = "direct", 0
        r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0]
        assert rel(g.control, r.control) < 1e-11
        assert np.max(np.abs(g.record.objectives() - r.record.objectives())) < 1e-11
    finally:
        c.close()


@pytest.mark.slow
@pytest.mark.parametrize("tag", ["literal", "fast"])
def test_ising10_config3_blocked(ctx, tag):
    # BASELINE config 3 at full size sharded into 8 blocks (the 8-GPU layout, emulated on one
    # device), 20 outer iterations at both step sizes, against the oracle's frozen direct-plan
    # outputs (tests/golden/make_baseline_fixtures.py)
    fx = np.load(FIXTURES / "config3_full.npz")
    w = problems.ising10(iterations=20)
    w.config.plan, w.config.blocks = "assembled", 8
    w.solver.step_size = float(fx[f"{tag}_rho"])
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    compare_run(g, fx, tag, u0=w.u0)


@pytest.mark.slow
def test_ising10_config3_reference_assembled_chain(ctx):
    # blocks = L = 256: the reference's assembled plan (one 1024 x 1024 propagator per
    # subinterval, chained), 2 iterations against the frozen direct-plan fixture's first records
    fx = np.load(FIXTURES / "config3_full.npz")
    w = problems.ising10(iterations=2)
    w.config.plan, w.config.blocks = "assembled", w.config.subintervals
    w.solver.step_size = float(fx["fast_rho"])
    g = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
    assert np.max(np.abs(g.record.objectives() - fx["fast_objective"][:3])) < 1e-10
    tv = np.array([it.task_values for it in g.record.iterations])
    assert np.max(np.abs(tv - fx["fast_task_values"][:3])) < 1e-10

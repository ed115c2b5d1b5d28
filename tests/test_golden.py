"""Golden vectors (tests/golden/*.npz, made by tests/golden/make_golden.py from the pinned
oracle): the CPU oracle must keep reproducing them (checker drift), and the device library
must match them within north_star's fp64 tolerances (controls rel 1e-9, objectives 1e-10)."""
from pathlib import Path

import numpy as np
import pytest

from paper_1603_01237_b200 import ism as I
from tests import oracle_api as O
from tests.golden.cases import CASES

GOLDEN = Path(__file__).parent / "golden"


def load(name):
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_reproduces_golden(name):
    w, arith = CASES[name]()
    g = load(name)
    runs = O.ism_run(w.problem, w.u0, w.config, w.solver, arith)
    ctl = np.stack([r.control for r in runs])
    obj = np.stack([r.record.objectives() for r in runs])
    assert np.max(np.abs(ctl - g["control"])) <= 1e-12 * max(1.0, np.max(np.abs(g["control"])))
    assert np.max(np.abs(obj - g["objective"])) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_device_matches_golden(ctx, name):
    w, _ = CASES[name]()
    g = load(name)
    runs = I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
    ctl = np.stack([r.control for r in runs])
    obj = np.stack([r.record.objectives() for r in runs])
    ex = np.stack([np.array([np.nan if it.exact_objective is None else it.exact_objective
                             for it in r.record.iterations]) for r in runs])
    assert np.max(np.abs(ctl - g["control"])) / np.max(np.abs(g["control"])) <= 1e-9
    assert np.max(np.abs(obj - g["objective"])) <= 1e-10
    assert np.allclose(ex, g["exact"], rtol=0, atol=1e-10, equal_nan=True)

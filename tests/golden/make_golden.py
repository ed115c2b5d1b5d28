"""Regenerates tests/golden/*.npz from the CPU oracle (oracle/oracle.cpp), itself pinned to the
reference's compiled run_ism (tests/test_reference_pinning.py) and its known answers
(tests/test_oracle_kats.py).  The vectors freeze the checker (CPU tests) and let the GPU tests
run without re-running long oracle jobs.  The condensate case starts from the stationary states
of problems.stationary_state, which agree with the reference's ground_state to 1e-11
(test_stationary_state_matches_reference_ground_state).

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from tests.golden.cases import CASES  # noqa: E402
from tests import oracle_api as O  # noqa: E402


def main():
    for name, make in CASES.items():
        w, arith = make()
        runs = O.ism_run(w.problem, w.u0, w.config, w.solver, arith)
        ctl = np.stack([r.control for r in runs])
        obj = np.stack([r.record.objectives() for r in runs])
        err = np.stack([np.array([np.nan if it.error is None else it.error for it in r.record.iterations])
                        for r in runs])
        ex = np.stack([np.array([np.nan if it.exact_objective is None else it.exact_objective
                                 for it in r.record.iterations]) for r in runs])
        np.savez_compressed(Path(__file__).parent / f"{name}.npz", control=ctl, objective=obj, error=err,
                            exact=ex)
        print(name, ctl.shape, obj[:, -1])


if __name__ == "__main__":
    main()

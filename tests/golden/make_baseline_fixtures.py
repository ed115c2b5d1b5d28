"""Oracle outputs of the full-size BASELINE configs 3 and 4 at the north_star iteration counts,
frozen as fixtures so the GPU suite compares against them without re-running hour-scale CPU
jobs on the GPU box (VERDICT r01 "parity at the north_star bar"):

* config 3 (ising10: d = 1024, K = 4000, L = 256): 20 outer iterations at rho = 0.1 and at
  rho = 0.1/dt -- controls (2 x 4000), objective and residual histories;
* config 4 (gpe1024: 1024 points, K = 10000, L = 64, split variant): 100 outer iterations at
  rho = 0.1 and rho = 0.1/dt with the exact payoff logged -- controls, objective, exact payoff
  and residual histories.

The checker is the CPU oracle (oracle/oracle.cpp, test infrastructure), structured Cayley
arithmetic for config 3 (pinned against the dense-LU reference arithmetic in
tests/test_oracle_kats.py), split-step Fourier for config 4.

    python tests/golden/make_baseline_fixtures.py [config3] [config4]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_1603_01237_b200 import problems  # noqa: E402
from tests import oracle_api as O  # noqa: E402

OUT = Path(__file__).parent


def build(name: str, fast: bool):
    if name == "config3":
        w = problems.ising10(iterations=20)
    else:
        w = problems.gpe1024(iterations=100)
        w.config.log_exact_objective = True
    if fast:
        w.solver.step_size = w.rho_fast
    return w


def run(name: str):
    out = {}
    for fast in (False, True):
        w = build(name, fast)
        t0 = time.time()
        r = O.ism_run(w.problem, w.u0, w.config, w.solver, O.STRUCTURED)[0]
        its = r.record.iterations
        tag = "fast" if fast else "literal"
        out[f"{tag}_control"] = r.control
        out[f"{tag}_objective"] = r.record.objectives()
        out[f"{tag}_error"] = np.array([np.nan if it.error is None else it.error for it in its])
        out[f"{tag}_exact"] = np.array([np.nan if it.exact_objective is None else it.exact_objective for it in its])
        out[f"{tag}_task_values"] = np.array([it.task_values for it in its])
        out[f"{tag}_rho"] = np.array(w.solver.step_size)
        if name == "config4":  # host-dependent iterative eigen-solve: freeze the states used
            out["initial"], out["target"] = np.asarray(w.problem.initial), np.asarray(w.problem.target)
        print(name, tag, f"{time.time() - t0:.1f}s", "final objective", out[f"{tag}_objective"][-1], flush=True)
    np.savez_compressed(OUT / f"{name}_full.npz", **out)


if __name__ == "__main__":
    for name in (sys.argv[1:] or ["config3", "config4"]):
        run(name)

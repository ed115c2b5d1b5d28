"""Sensitivity of BASELINE config 4 (gpe1024, split variant, 100 outer iterations) to rounding.

Runs the device path at both step sizes from u0 and from u0 + eps, and prints, per
iteration, the objective difference against the oracle's frozen fixture next to the difference
the eps-perturbation alone produces.  When the two columns grow together, the gap to the
fixture is the iteration's own amplification of last-bit differences, not a kernel defect.
usage: python tools/config4_drift.py [eps]
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1603_01237_b200 import ism as I  # noqa: E402
from paper_1603_01237_b200 import problems  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def main():
    eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-12
    fx = np.load(ROOT / "tests" / "golden" / "config4_full.npz")
    out = {}
    for tag in ("literal", "fast"):
        runs = []
        for shift in (0.0, eps):
            w = problems.gpe1024(iterations=100)
            w.problem.initial, w.problem.target = fx["initial"], fx["target"]
            w.config.log_exact_objective = True
            w.solver.step_size = float(fx[f"{tag}_rho"])
            runs.append(I.run_ism(w.problem, np.asarray(w.u0) + shift, w.config, w.solver))
        g, gp = runs
        o, op, of = g.record.objectives(), gp.record.objectives(), fx[f"{tag}_objective"]
        rows = []
        for k in (0, 1, 2, 3, 5, 10, 20, 30, 50, 70, 100):
            rows.append({"k": k, "vs_fixture": float(abs(o[k] - of[k])), "vs_perturbed": float(abs(op[k] - o[k]))})
            print(tag, rows[-1], flush=True)
        out[tag] = {
            "eps": eps,
            "control_rel_vs_fixture": rel(g.control, fx[f"{tag}_control"]),
            "control_rel_vs_perturbed": rel(gp.control, g.control),
            "rows": rows,
        }
        print(tag, {k: v for k, v in out[tag].items() if k != "rows"}, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

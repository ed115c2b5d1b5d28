"""Parallel efficiency vs L for BASELINE config 2 (rotor j <= 20, K = 20000) on the B200, with
the reference's own definitions (efficiency_table / time_to_target, runtime.cpp:117-153, and the
`qoc bench` CSV of tools/main.cpp:304-375): t(eps, L) = cumulative device time per outer
iteration until the objective is within eps of the best L = 1 objective; S = t(eps,1)/t(eps,L),
Eff = 100 S / L.  ISM iterates are L-invariant (Theorem 2), so the L runs follow the same
objective history and the table measures how well the device turns subintervals into speed.

    python tools/efficiency_vs_L.py [ITERATIONS] [OUT_DIR] [rotor21|spins]

`spins` is the paper's own efficiency experiment: the 5-spin
density-matrix problem, gradient solver, rho = 1e4, Crank-Nicolson with dt = T / 2^15, at
eps = 0.32, 0.89, 1.74 -- here for L = 1 ... 256 subintervals on one GPU.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1603_01237_b200 import _native, problems, wire  # noqa: E402
from paper_1603_01237_b200 import ism as I  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 600
    out = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out" / "efficiency"
    out.mkdir(parents=True, exist_ok=True)
    name = sys.argv[3] if len(sys.argv) > 3 else "rotor21"
    ctx = _native.default_context()
    runs, summary = [], []
    for L in ((1, 2, 4, 8, 16, 32, 64, 128, 256) if name == "spins" else (1, 8, 32, 128)):
        if name == "spins":
            w = problems.spins_preset(quick=False, subintervals=L, iterations=iters)
        else:
            w = problems.rotor21(subintervals=L, iterations=iters)
            w.solver.step_size = w.rho_fast
        I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)  # warm (context, graph cache)
        r = I.run_ism(w.problem, w.u0, w.config, w.solver, ctx)
        runs.append((L, r.record))
        its = r.record.iterations[1:]
        summary.append({"L": L, "iterations": len(its), "ms_per_iteration": 1e3 * sum(i.device_seconds for i in its) / len(its),
                        "final_objective": r.record.iterations[-1].objective})
    eps = [0.32, 0.89, 1.74] if name == "spins" else [0.1, 0.01, 0.001]
    csv = wire.bench_efficiency_csv(runs, eps)
    (out / f"efficiency_{name}.csv").write_text(csv)
    (out / f"efficiency_{name}.json").write_text(json.dumps({"workload": name, "rho": "1e4 (preset)" if name == "spins" else "0.1/dt",
                                                             "runs": summary, "eps": eps, "csv": csv}, indent=1))
    print(csv)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()

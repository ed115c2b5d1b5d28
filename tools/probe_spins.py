"""Device time per outer iteration of the reference's `spins` preset at full size (5 spins:
32 x 32 density matrices, 10 controls, 2^15 steps; the paper's headline physical case) for a few
subinterval counts, and the oracle's time for one iteration of the same problem."""
import json, sys, time
sys.path.insert(0, '.')
from paper_1603_01237_b200 import ism as I, problems
from tests import oracle_api as O

out = {}
for L in (16, 64, 256):
    w = problems.spins_preset(quick=False, subintervals=L, iterations=3)
    t0 = time.time()
    r = I.run_ism(w.problem, w.u0, w.config, w.solver)
    secs = [it.device_seconds for it in r.record.iterations]
    out[f"L{L}"] = {"wall": time.time() - t0, "bootstrap_s": secs[0], "iteration_s": secs[1:],
                    "steps_per_s": 2 * w.problem.grid.steps / (sum(secs[1:]) / len(secs[1:]))}
    print(json.dumps({f"L{L}": out[f"L{L}"]}), flush=True)
if len(sys.argv) > 1 and sys.argv[1] == "cpu":
    w = problems.spins_preset(quick=False, subintervals=64, iterations=1)
    t0 = time.time()
    O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE)
    print(json.dumps({"oracle_L64_one_iteration_wall_s": time.time() - t0}), flush=True)

"""Run one workload for a few outer iterations (for ncu launch lists / captures)."""
import sys, time, json
sys.path.insert(0, '.')
from bench import build_workload
from paper_1603_01237_b200 import ism as I
name = sys.argv[1]; it = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = build_workload(name, it, 0, 1)
if name == "batch4096" and len(sys.argv) > 3:
    from paper_1603_01237_b200 import problems
    w = problems.batch4096(batch=int(sys.argv[3]), iterations=it); w.solver.step_size = w.rho_fast
t = time.time(); r = I.run_ism_batch(w.problem, w.u0, w.config, w.solver)
print(json.dumps({"workload": name, "wall": time.time() - t, "device_seconds": [x.device_seconds for x in r[0].record.iterations]}))

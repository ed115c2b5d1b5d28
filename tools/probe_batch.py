"""Timing probe: BASELINE config 5 (4096 x d=16) on the device for a few iterations."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
from paper_1603_01237_b200 import problems, ism as I
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
it = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t = time.time(); w = problems.batch4096(batch=B, iterations=it); print('gen', time.time() - t, flush=True)
t = time.time(); runs = I.run_ism_batch(w.problem, w.u0, w.config, w.solver); wall = time.time() - t
secs = [x.device_seconds for x in runs[0].record.iterations]
print(json.dumps({"B": B, "wall": wall, "device_seconds": secs}))
steps = 2 * 2000 * B
print("steps/s per iteration:", [steps / s for s in secs[1:]])

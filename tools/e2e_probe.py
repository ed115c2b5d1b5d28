"""Host-side breakdown of one run_ism_batch call (QOC_TRACE_HOST phases from the driver plus the
Python packing/unpacking), for the e2e leg of bench.py:  python tools/e2e_probe.py WORKLOAD K"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["QOC_TRACE_HOST"] = "1"
import bench  # noqa: E402
from paper_1603_01237_b200 import _native  # noqa: E402
from paper_1603_01237_b200 import ism as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "batch4096"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = _native.default_context()
w = bench.build_workload(name, K, 0, 1)
I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
for _ in range(2):
    t0 = time.perf_counter()
    packed = I.pack_problem(w.problem)
    t1 = time.perf_counter()
    I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
    t2 = time.perf_counter()
    print(f"[py] pack {1e3 * (t1 - t0):.1f} ms, call {1e3 * (t2 - t1):.1f} ms", file=sys.stderr, flush=True)

import os, time, sys
sys.path.insert(0, '.')
os.environ['QOC_TRACE_HOST'] = '1'
from paper_1603_01237_b200 import ism as I, problems, _native
ctx = _native.default_context()
w = problems.batch4096(iterations=5); w.solver.step_size = w.rho_fast
I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx)
for _ in range(2):
    t = time.perf_counter(); I.run_ism_batch(w.problem, w.u0, w.config, w.solver, ctx); print('call', time.perf_counter() - t, file=sys.stderr)

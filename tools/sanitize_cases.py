"""Small cases that drive every device code path once, for compute-sanitizer (memcheck /
racecheck / synccheck): the smoke workloads plus the Neumann/tensor-core config-5 sweep and its
streaming evaluation, the cluster node sweeps of the d = 1024 spin register, the d = 48 dense
CTA kernels and the density-matrix kind."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_1603_01237_b200 import ism as I  # noqa: E402
from paper_1603_01237_b200 import problems  # noqa: E402
from tests import oracle_api as O  # noqa: E402

__graft_entry__.smoke()
w = problems.batch4096(batch=9, iterations=2)  # dense_nm_* + dense_pc_eval16
I.run_ism_batch(w.problem, w.u0, w.config, w.solver)
w = problems.ising10(steps=64, T=0.48, iterations=1, subintervals=8)  # bitflip cluster sweeps
I.run_ism(w.problem, w.u0, w.config, w.solver)
p, u = O.dense_fixture(2650, dim=48, steps=6, channels=2, quadratic=True)  # dense_big
I.run_ism(p, u, I.IsmConfig(subintervals=2, max_outer=2, eta=0.0), I.SolverSpec(step_size=0.5))
w = problems.spins_preset(quick=True, iterations=2, steps=64)  # density kind
I.run_ism(w.problem, w.u0, w.config, w.solver)
print("sanitize cases done")

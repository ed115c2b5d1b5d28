"""Host-side logic that needs no GPU: the solver spec packing, the inner-solver event strings,
the basis form of the condensate potentials, and the new C-ABI symbols."""
import ctypes as C

import numpy as np

from paper_1603_01237_b200 import abi
from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200.models import BasisCondensateModel, CondensateModel


def test_solver_spec_packs_the_reference_defaults():
    s = I.pack_solver(I.SolverSpec(kind="newton"))  # optimizers.hpp:9-30
    assert s.kind == abi.SOLVER_NEWTON and s.inner_iterations == 1
    assert (s.fixed_point_tol, s.fixed_point_max_iter) == (1e-12, 50)
    assert (s.gmres_restart, s.gmres_max_iter, s.gmres_tol, s.hvp_scale) == (30, 200, 1e-6, 1e-5)
    assert I.pack_solver(I.SolverSpec(kind="monotonic")).kind == abi.SOLVER_MONOTONIC


def test_solver_events_wording():
    # ism.cpp:503-511: per task, the guard event before the fallback event
    stats = np.array([[0, 3, 0], [1, 2, 0], [7, 9, 4]], dtype=np.int32)
    assert I.solver_events(stats) == [
        "task 0: 1 Newton directions replaced by gradient steps",
        "task 1: kept 3 slices at previous values",
        "task 1: 2 Newton directions replaced by gradient steps",
    ]


def test_basis_form_of_the_lattice_potential():
    lat = CondensateModel(64, -16.0, 16.0, abi.POT_LATTICE, [1.0, 5.0, 1.0], 10.0)
    bas = BasisCondensateModel.lattice(64, -16.0, 16.0, 1.0, 5.0, 1.0, 10.0)
    for u in (-0.7, 0.0, 0.3, 2.5):
        assert np.max(np.abs(lat.potential([u]) - bas.potential([u]))) < 1e-13
        dv = 5.0 * 1.0 * np.sin(2.0 * (lat.x - u))  # v0 k sin(2k(x - u))
        assert np.max(np.abs(bas.potential_derivative(0, [u]) - dv)) < 1e-13
    packed = I.pack_problem(I.ControlProblem(bas, I.TimeGrid.over(0.0, 1.0, 4), np.ones(64), np.ones(64), None))
    assert packed is not None
    assert bas.basis.shape == (3, 64) and list(bas.term_type) == [abi.TERM_POWER, abi.TERM_COS, abi.TERM_SIN]


def test_power_terms_and_finite_difference_derivative():
    x = np.linspace(-1.0, 1.0, 16, endpoint=False)
    m = BasisCondensateModel(16, -1.0, 1.0, [(x * x, "power", 0), (x, "power", 1), (0.5 * x, "power", 3),
                                             (np.cos(x), "sin", 1.3)], 0.0)
    u, h = 0.37, 1e-6
    fd = (m.potential([u + h]) - m.potential([u - h])) / (2 * h)
    assert np.max(np.abs(fd - m.potential_derivative(0, [u]))) < 1e-8


def test_library_exports_the_round2_symbols():
    from paper_1603_01237_b200 import build
    lib = C.CDLL(str(build.OUT))
    for name in ("qoc_ctx_solver_stats", "qoc_imaginary_time", "qoc_comm_unique_id", "qoc_ctx_init_comm"):
        assert hasattr(lib, name), name

"""ctypes mirror of include/qoc_gpu.h (the C ABI of the device path).

The structs here are byte-for-byte the ones declared in ``include/qoc_gpu.h``; the
problem packer turns the Python mirror of the reference's ``ControlProblem``
(objective.hpp:18-24) into a ``qoc_problem_v1`` whose arrays stay alive as long as
the returned :class:`PackedProblem`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

QOC_ABI_VERSION = 2

QOC_OK, QOC_EINVAL, QOC_ELOGIC, QOC_ECUDA, QOC_ENCCL, QOC_ERUNTIME = range(6)
KIND_DENSE, KIND_TRIDIAG, KIND_BITFLIP, KIND_STRANG, KIND_DENSITY = range(5)
POT_TRAP, POT_LATTICE, POT_BASIS = range(3)
TERM_POWER, TERM_COS, TERM_SIN = range(3)
MAX_POT_TERMS = 8
VARIANT_INTERPOLATED, VARIANT_SPLIT = range(2)
PLAN_ASSEMBLED, PLAN_DIRECT = range(2)
PARTITION_BALANCED, PARTITION_UNIFORM, PARTITION_EXPLICIT = range(3)
SOLVER_GRADIENT, SOLVER_MONOTONIC, SOLVER_NEWTON = range(3)
FORM_OVERLAP, FORM_TRACKING = range(2)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class ProblemV1(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("kind", C.c_int32), ("dim", C.c_int32),
        ("channels", C.c_int32), ("steps", C.c_int32), ("batch", C.c_int32),
        ("t_start", C.c_double), ("dt", C.c_double), ("ip_weight", C.c_double),
        ("h0", _dp), ("linear", _dp), ("quadratic", _dp),
        ("tri_diag", _dp), ("tri_sub", _dp), ("tri_has_quadratic", C.c_int32),
        ("nspins", C.c_int32), ("bf_axis", _ip), ("bf_coef", _dp),
        ("kinetic", _dp), ("grid_x", _dp), ("potential", C.c_int32),
        ("pot_params", C.c_double * 4), ("kappa", C.c_double),
        ("pot_terms", C.c_int32), ("pot_reserved", C.c_int32),
        ("pot_term_type", _ip), ("pot_term_param", _dp), ("pot_basis", _dp),
        ("initial", _dp), ("target", _dp), ("penalty", _dp),
    ]


class IsmConfigV1(C.Structure):
    _fields_ = [
        ("subintervals", C.c_int32), ("workers", C.c_int32), ("max_outer", C.c_int32),
        ("variant", C.c_int32), ("plan", C.c_int32), ("compute_error", C.c_int32),
        ("log_exact_objective", C.c_int32), ("checkpoint_stride", C.c_int32),
        ("partition", C.c_int32), ("blocks", C.c_int32), ("eta", C.c_double),
        ("node_index", _ip),
    ]


class SolverV1(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("inner_iterations", C.c_int32),
        ("naive_nonlinear_adjoint", C.c_int32), ("checkpoint_stride", C.c_int32),
        ("step_size", C.c_double),
        ("fixed_point_tol", C.c_double), ("fixed_point_max_iter", C.c_int32),
        ("gmres_restart", C.c_int32), ("gmres_max_iter", C.c_int32), ("reserved", C.c_int32),
        ("gmres_tol", C.c_double), ("hvp_scale", C.c_double),
    ]


class IterRecordV1(C.Structure):
    _fields_ = [
        ("iteration", C.c_int32), ("has_error", C.c_int32), ("has_exact_objective", C.c_int32),
        ("reserved", C.c_int32), ("objective", C.c_double), ("exact_objective", C.c_double),
        ("error", C.c_double), ("device_seconds", C.c_double),
    ]


class RunStatusV1(C.Structure):
    _fields_ = [("aborted", C.c_int32), ("iterations_recorded", C.c_int32),
                ("abort_reason", C.c_char * 240)]


class ProfileV1(C.Structure):
    _fields_ = [("task_launches", C.c_int64), ("task_ms", C.c_double), ("other_launches", C.c_int64),
                ("other_ms", C.c_double), ("iterations", C.c_int64), ("iteration_ms", C.c_double),
                ("iteration_launches", C.c_int64)]


OPT_PROFILE, OPT_FLUSH_L2_BYTES = 1, 2
COMM_ID_BYTES = 128


class CtxOptsV1(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("device", C.c_int32), ("reserved", C.c_int32 * 6)]


REC_DTYPE = np.dtype([
    ("iteration", "<i4"), ("has_error", "<i4"), ("has_exact_objective", "<i4"), ("reserved", "<i4"),
    ("objective", "<f8"), ("exact_objective", "<f8"), ("error", "<f8"), ("device_seconds", "<f8"),
])
assert REC_DTYPE.itemsize == C.sizeof(IterRecordV1)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def cplx(a) -> np.ndarray:
    """complex array -> contiguous interleaved float64 (re, im) view, Eigen byte order."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a.view(np.float64).reshape(-1)


@dataclass
class PackedProblem:
    """A qoc_problem_v1 plus the numpy buffers it points into."""
    struct: ProblemV1
    keep: list = field(default_factory=list)

    @property
    def ref(self):
        return C.byref(self.struct)


def colmajor(m: np.ndarray) -> np.ndarray:
    """numpy (..., d, d) matrices -> column-major storage order (Eigen layout)."""
    return np.ascontiguousarray(np.swapaxes(np.asarray(m), -1, -2))

"""ctypes wrapper of the CPU oracle (oracle/_build/liboracle.so) -- TEST INFRASTRUCTURE.

The oracle restates the reference's ISM path on the CPU (oracle/oracle.cpp).  It takes the
same packed qoc_problem_v1 as the device library, so a test packs a problem once and feeds
both sides.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_1603_01237_b200 import abi
from paper_1603_01237_b200 import ism as I

ROOT = Path(__file__).resolve().parents[1]
LIBPATH = ROOT / "oracle" / "_build" / "liboracle.so"
REFERENCE, STRUCTURED = 0, 1

_lib = None


def lib():
    global _lib
    if _lib is None:
        # make is a no-op when the library is newer than oracle.cpp / oracle.h / qoc_gpu.h
        if not LIBPATH.exists() or __import__("shutil").which("make"):
            subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=not LIBPATH.exists())
        _lib = C.CDLL(str(LIBPATH))
        _lib.oracle_ism_run.restype = C.c_int32
    return _lib


def _err():
    return C.create_string_buffer(512)


def _check(code, err):
    I.raise_for(code, err.value.decode())


def ism_run(p: I.ControlProblem, u0, cfg: I.IsmConfig, solver: I.SolverSpec,
            arith: int = STRUCTURED, threads: int | None = None) -> list[I.IsmRun]:
    packed = I.pack_problem(p)
    B, Cn, K = p.batch, p.model.channels(), p.grid.steps
    u_in = I.controls_to_abi(u0, B, Cn, K)
    u_out = np.empty_like(u_in)
    c, keep = I.pack_config(cfg)
    s = I.pack_solver(solver)
    cap, recs, tvals, status = I.run_buffers(p, cfg)
    err = _err()
    threads = threads or os.cpu_count() or 1
    code = lib().oracle_ism_run(packed.ref, C.byref(c), C.byref(s), abi.dptr(u_in), abi.dptr(u_out),
                                recs.ctypes.data_as(C.c_void_p), C.c_int32(cap), abi.dptr(tvals),
                                status, C.c_int32(arith), C.c_int32(threads), err, C.c_size_t(512))
    _check(code, err)
    u = I.controls_from_abi(u_out, B, Cn, K)
    L = cfg.subintervals

    def stats(b, k):
        row = np.zeros((3, L), dtype=np.int32)
        ok = lib().oracle_solver_stats(C.c_int32(b), C.c_int32(k), C.c_int32(L), row.ctypes.data_as(C.c_void_p))
        return row if ok == abi.QOC_OK else None
    runs = I.unpack_all(recs, tvals, status, cfg, solver, stats=stats if solver.kind != "gradient" else None)
    for r in runs:
        _ = r.iterations  # build now: the counters belong to this call
    return [I.IsmRun(u[b], r) for b, r in enumerate(runs)]


def propagate_final(p, u, arith=STRUCTURED):
    packed = I.pack_problem(p)
    B, d = p.batch, int(np.prod(I.state_shape(p.model)))
    u_in = I.controls_to_abi(u, B, p.model.channels(), p.grid.steps)
    out = np.empty(2 * B * d)
    err = _err()
    _check(lib().oracle_propagate_final(packed.ref, abi.dptr(u_in), abi.dptr(out), C.c_int32(arith),
                                        err, C.c_size_t(512)), err)
    return I.unpack_states(out, p.model, (B,))


def propagate(p, u, arith=STRUCTURED):
    packed = I.pack_problem(p)
    B, d, K = p.batch, p.model.state_dim(), p.grid.steps
    u_in = I.controls_to_abi(u, B, p.model.channels(), K)
    out = np.empty(2 * B * (K + 1) * d)
    err = _err()
    _check(lib().oracle_propagate(packed.ref, abi.dptr(u_in), abi.dptr(out), C.c_int32(arith), err,
                                  C.c_size_t(512)), err)
    return out.view(np.complex128).reshape(B, K + 1, d)


def objective_gradient(p, u, form="tracking", naive=False, stride=0, arith=STRUCTURED):
    packed = I.pack_problem(p)
    B, Cn, K = p.batch, p.model.channels(), p.grid.steps
    u_in = I.controls_to_abi(u, B, Cn, K)
    val = np.empty(B)
    grad = np.empty_like(u_in)
    f = abi.FORM_OVERLAP if form == "overlap" else abi.FORM_TRACKING
    err = _err()
    _check(lib().oracle_objective_gradient(packed.ref, abi.dptr(u_in), C.c_int32(f), C.c_int32(int(naive)),
                                           C.c_int32(stride), abi.dptr(val), abi.dptr(grad),
                                           C.c_int32(arith), err, C.c_size_t(512)), err)
    return val, I.controls_from_abi(grad, B, Cn, K)


def assemble_propagator(p, u, arith=STRUCTURED):
    packed = I.pack_problem(p)
    B, d = p.batch, p.model.state_dim()
    u_in = I.controls_to_abi(u, B, p.model.channels(), p.grid.steps)
    out = np.empty(2 * B * d * d)
    err = _err()
    _check(lib().oracle_assemble_propagator(packed.ref, abi.dptr(u_in), abi.dptr(out), C.c_int32(arith),
                                            err, C.c_size_t(512)), err)
    return np.swapaxes(out.view(np.complex128).reshape(B, d, d), 1, 2)


def step(p, u_col, dt, state, adjoint=False, psi_j=None, naive=False, arith=STRUCTURED):
    packed = I.pack_problem(p)
    d = p.model.state_dim()
    uc = np.ascontiguousarray(np.asarray(u_col, dtype=np.float64).reshape(-1))
    sin = abi.cplx(np.asarray(state).reshape(-1))
    pj = abi.cplx(np.asarray(psi_j).reshape(-1)) if psi_j is not None else None
    out = np.empty(2 * d)
    err = _err()
    _check(lib().oracle_step(packed.ref, abi.dptr(uc), C.c_double(dt), abi.dptr(sin), abi.dptr(pj),
                             C.c_int32(int(adjoint)), C.c_int32(int(naive)), abi.dptr(out),
                             C.c_int32(arith), err, C.c_size_t(512)), err)
    return out.view(np.complex128).copy()


def dft(x, inverse=False):
    xi = abi.cplx(x)
    out = np.empty_like(xi)
    assert lib().oracle_dft(C.c_int32(len(x)), abi.dptr(xi), abi.dptr(out), C.c_int32(int(inverse))) == 0
    return out.view(np.complex128).copy()


def verify_decomposition(p, u, parts, arith=STRUCTURED):
    packed = I.pack_problem(p)
    u_in = I.controls_to_abi(u, 1, p.model.channels(), p.grid.steps)
    fm, gm = C.c_double(), C.c_double()
    err = _err()
    _check(lib().oracle_verify_decomposition(packed.ref, abi.dptr(u_in), C.c_int32(parts), C.byref(fm),
                                             C.byref(gm), C.c_int32(arith), err, C.c_size_t(512)), err)
    return fm.value, gm.value


def boundary_sweep(p, u, nodes, arith=STRUCTURED):
    packed = I.pack_problem(p)
    d = p.model.state_dim()
    u_in = I.controls_to_abi(u, 1, p.model.channels(), p.grid.steps)
    L = len(nodes) - 1
    ni = np.ascontiguousarray(nodes, dtype=np.int32)
    ps = np.empty(2 * (L + 1) * d)
    cs = np.empty(2 * (L + 1) * d)
    err = _err()
    _check(lib().oracle_boundary_sweep(packed.ref, abi.dptr(u_in), C.c_int32(L), abi.iptr(ni), abi.dptr(ps),
                                       abi.dptr(cs), C.c_int32(arith), err, C.c_size_t(512)), err)
    return ps.view(np.complex128).reshape(L + 1, d), cs.view(np.complex128).reshape(L + 1, d)


def dense_fixture(seed, dim=4, steps=16, channels=2, quadratic=False, alpha=0.1, duration=1.0,
                  control_amplitude=0.8, random_penalty=False):
    """fixtures::dense_fixture (fixtures.hpp:66-112), vector kind, same mt19937 draws."""
    dd = dim * dim
    h0 = np.empty(2 * dd)
    lin = np.empty(2 * dd * channels)
    quad = np.empty(2 * dd * channels) if quadratic else np.empty(2)
    ini, tgt = np.empty(2 * dim), np.empty(2 * dim)
    pen = np.empty(steps)
    ctl = np.empty(channels * steps)
    lib().oracle_dense_fixture(C.c_uint32(seed), dim, steps, channels, int(quadratic), C.c_double(alpha),
                               int(random_penalty), C.c_double(control_amplitude), abi.dptr(h0),
                               abi.dptr(lin), abi.dptr(quad), abi.dptr(ini), abi.dptr(tgt),
                               abi.dptr(pen), abi.dptr(ctl))

    def mats(buf, n):
        return np.swapaxes(buf.view(np.complex128).reshape(n, dim, dim), 1, 2)

    from paper_1603_01237_b200.models import DenseModel
    model = DenseModel(mats(h0, 1)[0], mats(lin, channels), mats(quad, channels) if quadratic else None)
    grid = I.TimeGrid.over(0.0, duration, steps)
    problem = I.ControlProblem(model, grid, ini.view(np.complex128).copy(), tgt.view(np.complex128).copy(),
                               pen)
    control = ctl.reshape(steps, channels).T.copy()
    return problem, control


def strang_fixture(seed, points=24, x_min=-8.0, x_max=8.0, distance=6.0, kappa=1.0, steps=12,
                   duration=0.5, alpha=0.05, control_amplitude=0.9):
    """fixtures::strang_fixture (fixtures.hpp:208-234)."""
    from paper_1603_01237_b200.models import CondensateModel
    ini, tgt, ctl = np.empty(2 * points), np.empty(2 * points), np.empty(steps)
    lib().oracle_strang_fixture(C.c_uint32(seed), points, C.c_double(x_min), C.c_double(x_max), steps,
                                C.c_double(control_amplitude), abi.dptr(ini), abi.dptr(tgt), abi.dptr(ctl))
    model = CondensateModel(points, x_min, x_max, abi.POT_TRAP, [distance], kappa)
    grid = I.TimeGrid.over(0.0, duration, steps)
    problem = I.ControlProblem(model, grid, ini.view(np.complex128).copy(), tgt.view(np.complex128).copy(),
                               np.full(steps, alpha))
    return problem, ctl.reshape(1, steps)


class Rng:
    """std::mt19937-driven draws of the reference tests (random_cvec/state/hermitian)."""

    def __init__(self, seed):
        self.buf = C.create_string_buffer(5000)
        self.seed = seed
        self.fresh = True

    def _draw(self, what, n, scale, size):
        out = np.empty(2 * size)
        lib().oracle_rng(self.buf, int(self.fresh), C.c_uint32(self.seed), what, n, C.c_double(scale),
                         abi.dptr(out))
        self.fresh = False
        return out.view(np.complex128).copy()

    def cvec(self, n):
        return self._draw(0, n, 1.0, n)

    def state(self, n):
        return self._draw(1, n, 1.0, n)

    def hermitian(self, n, scale=1.0):
        return self._draw(2, n, scale, n * n).reshape(n, n).T.copy()


# ---- the reference itself (oracle/_ref/libqocref.so: /root/reference's run_ism compiled
# against the Eigen-subset shim by `make -C oracle ref`; absent on the GPU box) ------------------
REF_LIBPATH = ROOT / "oracle" / "_ref" / "libqocref.so"
_ref = None


def ref_available() -> bool:
    if Path("/root/reference/proj/core/src/ism.cpp").exists():  # up to date with ref_capi.cpp and the headers
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=not REF_LIBPATH.exists())
    return REF_LIBPATH.exists()


def ref_ism_run(p: I.ControlProblem, u0, cfg: I.IsmConfig, solver: I.SolverSpec) -> list[I.IsmRun]:
    """qoc::run_ism of the reference (ism.cpp:211-612), one problem at a time."""
    global _ref
    if _ref is None:
        _ref = C.CDLL(str(REF_LIBPATH))
        _ref.ref_ism_run.restype = C.c_int32
    packed = I.pack_problem(p)
    B, Cn, K = p.batch, p.model.channels(), p.grid.steps
    u_in = I.controls_to_abi(u0, B, Cn, K)
    u_out = np.empty_like(u_in)
    c, keep = I.pack_config(cfg)
    s = I.pack_solver(solver)
    cap, recs, tvals, status = I.run_buffers(p, cfg)
    err = _err()
    code = _ref.ref_ism_run(packed.ref, C.byref(c), C.byref(s), abi.dptr(u_in), abi.dptr(u_out),
                            recs.ctypes.data_as(C.c_void_p), C.c_int32(cap), abi.dptr(tvals), status, err,
                            C.c_size_t(512))
    _check(code, err)
    u = I.controls_from_abi(u_out, B, Cn, K)
    runs = I.unpack_all(recs, tvals, status, cfg, solver)
    for b, r in enumerate(runs):  # the reference's own IterationStat::events
        for k, it in enumerate(r.iterations):
            buf = C.create_string_buffer(1 << 16)
            if _ref.ref_iteration_events(C.c_int32(b), C.c_int32(k), buf, C.c_size_t(len(buf))) == abi.QOC_OK:
                ev = [e for e in buf.value.decode().split("\n") if e]
                if r.aborted and k == len(r.iterations) - 1:
                    ev = [e for e in ev if e != r.abort_reason]
                    it.events[:0] = ev
                else:
                    it.events.extend(ev)
    return [I.IsmRun(u[b], r) for b, r in enumerate(runs)]


def basis_fixture(seed, points=32, steps=16, duration=0.4, kappa=1.5, alpha=0.05):
    """A caller-defined condensate potential through the basis plugin (QOC_POT_BASIS): a breathing,
    tilted trap in a modulated lattice,
        V(x, u) = x^2/2 + 0.3 x u + 0.05 x^2 u^2 + 1.2 cos^2(0.8 (x - u)),
    with states and control drawn like fixtures::strang_fixture."""
    from paper_1603_01237_b200.models import BasisCondensateModel
    x_min, x_max = -8.0, 8.0
    x = x_min + np.arange(points) * ((x_max - x_min) / points)
    k, v0 = 0.8, 1.2
    terms = [(0.5 * x * x + 0.5 * v0, "power", 0), (0.3 * x, "power", 1), (0.05 * x * x, "power", 2),
             (0.5 * v0 * np.cos(2 * k * x), "cos", 2 * k), (0.5 * v0 * np.sin(2 * k * x), "sin", 2 * k)]
    model = BasisCondensateModel(points, x_min, x_max, terms, kappa)
    ini, tgt, ctl = np.empty(2 * points), np.empty(2 * points), np.empty(steps)
    lib().oracle_strang_fixture(C.c_uint32(seed), points, C.c_double(x_min), C.c_double(x_max), steps,
                                C.c_double(0.9), abi.dptr(ini), abi.dptr(tgt), abi.dptr(ctl))
    grid = I.TimeGrid.over(0.0, duration, steps)
    problem = I.ControlProblem(model, grid, ini.view(np.complex128).copy(), tgt.view(np.complex128).copy(),
                               np.full(steps, alpha))
    return problem, ctl.reshape(1, steps)


def ref_ground_state(points, x_min, x_max, distance, kappa, u_frozen, imaginary_dt=1e-2, energy_tol=1e-10,
                     max_iterations=200000):
    """qoc::ground_state of the reference itself (models.cpp:129-294) on a TrappedCondensateModel:
    (psi, energy, chemical_potential, residual, iterations)."""
    global _ref
    if _ref is None:
        _ref = C.CDLL(str(REF_LIBPATH))
        _ref.ref_ism_run.restype = C.c_int32
    psi, sc = np.empty(2 * points), np.empty(4)
    code = _ref.ref_ground_state(C.c_int32(points), C.c_double(x_min), C.c_double(x_max), C.c_double(distance),
                                 C.c_double(kappa), C.c_double(u_frozen), C.c_double(imaginary_dt),
                                 C.c_double(energy_tol), C.c_int32(max_iterations), abi.dptr(psi), abi.dptr(sc))
    assert code == abi.QOC_OK
    return psi.view(np.complex128).copy(), sc[0], sc[1], sc[2], int(sc[3])

"""Reference-facing API of the ISM hot path (the Python mirror of qoc's C++ solver API).

    IsmRun run_ism(const ControlProblem&, const ControlField& u0, const IsmConfig&,
                   const SolverSpec&)                      -- ism.hpp:80-81, ism.cpp:211-612

``run_ism`` here has the same argument meaning, record semantics and error behaviour, and
executes on the B200 through ``libqoc_b200.so`` (include/qoc_gpu.h).  There is no CPU path:
if the native library is missing the call fails loudly (see ``_native``).

Controls are numpy arrays of shape (C, K) -- the reference's C x K sample matrix
(controls.hpp:33-60) -- or (B, C, K) for a batch of independent problems.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import abi
from .models import HamiltonianModel


# ----------------------------------------------------------------------------------------
# Exceptions mirroring the reference's exception types (SURVEY §8(b) conventions).
# ----------------------------------------------------------------------------------------
class InvalidArgument(ValueError):
    """std::invalid_argument"""


class LogicError(Exception):
    """std::logic_error"""


class QocRuntimeError(RuntimeError):
    """std::runtime_error (e.g. decomposition errors, controls.cpp:16-18)"""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure"""


def raise_for(code: int, msg: str) -> None:
    if code == abi.QOC_OK:
        return
    exc = {abi.QOC_EINVAL: InvalidArgument, abi.QOC_ELOGIC: LogicError,
           abi.QOC_ERUNTIME: QocRuntimeError}.get(code, DeviceError)
    raise exc(msg or f"qoc error {code}")


# ----------------------------------------------------------------------------------------
# Problem / config types
# ----------------------------------------------------------------------------------------
@dataclass(frozen=True)
class TimeGrid:
    """Uniform step grid (controls.hpp:14-25)."""
    t_start: float
    dt: float
    steps: int

    @staticmethod
    def over(t0: float, t1: float, steps: int) -> "TimeGrid":  # controls.cpp:55-59
        if steps <= 0:
            raise QocRuntimeError("TimeGrid: steps must be positive")
        if not t1 > t0:
            raise QocRuntimeError("TimeGrid: t_end must exceed t_start")
        return TimeGrid(float(t0), (t1 - t0) / steps, int(steps))

    def node(self, j: int) -> float:
        return self.t_start + self.dt * j


@dataclass
class ControlProblem:
    """objective.hpp:18-24: model, grid, initial and target states, per-step penalty."""
    model: HamiltonianModel
    grid: TimeGrid
    initial: np.ndarray            # (d,) or (B, d) complex
    target: np.ndarray             # (d,) or (B, d) complex
    penalty: Optional[np.ndarray] = None   # (K,) alpha_j, None = 0

    @property
    def batch(self) -> int:
        return self.model.batch


@dataclass
class IsmConfig:
    """ism.hpp:12-39 (plus the decomposition choice)."""
    subintervals: int = 1
    workers: int = 1
    eta: float = 1e-3
    max_outer: int = 50
    variant: str = "interpolated"      # or "split"
    plan: str = "assembled"            # or "direct"
    compute_error: bool = True
    log_exact_objective: bool = False
    checkpoint_stride: int = 0
    partition: str = "balanced"        # "uniform" = Decomposition::uniform; "explicit"
    node_index: Optional[Sequence[int]] = None
    # bit-flip kind, assembled plan: contiguous subinterval blocks of the blocked boundary
    # refresh (G = subintervals is the reference's per-subinterval chain); 0 = direct node
    # sweeps on one GPU, one block per rank under a communicator (qoc_gpu.h qoc_ctx_init_comm)
    blocks: int = 0


@dataclass
class SolverSpec:
    """optimizers.hpp:9-30.  kind is "gradient" (the hot path), "monotonic" or "newton"."""
    kind: str = "gradient"
    step_size: float = 1.0
    inner_iterations: int = 1
    naive_nonlinear_adjoint: bool = False
    checkpoint_stride: int = 0
    fixed_point_tol: float = 1e-12   # monotonic sweep: implicit per-slice update
    fixed_point_max_iter: int = 50
    gmres_restart: int = 30          # Newton direction: restarted GMRES on FD Hessian products
    gmres_max_iter: int = 200
    gmres_tol: float = 1e-6
    hvp_scale: float = 1e-5


@dataclass
class TaskStat:
    """runtime.hpp:38-42.  On the device every task of an iteration runs concurrently inside
    the same kernels: compute_seconds is the device time of the iteration's task kernels (an
    upper bound on each task), nothing is serialised (serialize_seconds = bytes_sent = 0)."""
    compute_seconds: float = 0.0
    serialize_seconds: float = 0.0
    bytes_sent: int = 0


@dataclass
class IterationStat:
    """runtime.hpp:44-63.  critical_path_seconds / wall_seconds are the device time of the
    iteration (CUDA events bracketing its launch sequence); events carry the reference's abort
    text at the iteration that stopped the run (ism.cpp:387,529-530,558)."""
    iteration: int
    objective: float
    exact_objective: Optional[float] = None
    error: Optional[float] = None
    task_values: list = field(default_factory=list)
    device_seconds: float = 0.0
    tasks: list = field(default_factory=list)
    events: list = field(default_factory=list)
    solver_stats: Optional[np.ndarray] = None  # [3][L] guard rejections, Newton fallbacks, GMRES iterations

    @property
    def critical_path_seconds(self) -> float:
        return self.device_seconds

    @property
    def wall_seconds(self) -> float:
        return self.device_seconds


class RunRecord:
    """runtime.hpp:65-75.  Records returned by a device run keep their per-iteration arrays and
    build the IterationStat list on first access of `iterations` (a 4096-problem batch returns
    ~10^5 of them; the e2e path should not pay for objects nobody reads)."""

    def __init__(self, subintervals: int = 1, workers: int = 1, solver: str = "gradient",
                 variant: str = "interpolated", plan: str = "assembled", iterations=None,
                 aborted: bool = False, abort_reason: str = ""):
        self.subintervals, self.workers, self.solver = subintervals, workers, solver
        self.variant, self.plan = variant, plan
        self.aborted, self.abort_reason = aborted, abort_reason
        self._iterations = list(iterations) if iterations is not None else []
        self._build = None

    @property
    def iterations(self) -> list:
        if self._build is not None:
            self._iterations, self._build = self._build(), None
        return self._iterations

    @iterations.setter
    def iterations(self, value) -> None:
        self._iterations, self._build = list(value), None

    def __repr__(self) -> str:
        return (f"RunRecord(subintervals={self.subintervals}, workers={self.workers}, solver={self.solver!r}, "
                f"variant={self.variant!r}, plan={self.plan!r}, iterations=<{len(self.iterations)}>, "
                f"aborted={self.aborted}, abort_reason={self.abort_reason!r})")

    def objectives(self) -> np.ndarray:
        return np.array([it.objective for it in self.iterations])

    def total_wall_seconds(self) -> float:  # runtime.cpp:104-108
        return float(sum(it.wall_seconds for it in self.iterations))

    def total_critical_path_seconds(self) -> float:  # runtime.cpp:110-114
        return float(sum(it.critical_path_seconds for it in self.iterations))


@dataclass
class IsmRun:
    """ism.hpp:74-77: the optimized control (C, K) and the run record."""
    control: np.ndarray
    record: RunRecord


# ----------------------------------------------------------------------------------------
# Packing into the C ABI (shared with the test-side oracle wrapper).
# ----------------------------------------------------------------------------------------
def _states(a, B: int, d: int, what: str, square: bool = False) -> np.ndarray:
    a = np.asarray(a, dtype=np.complex128)
    if square:  # d x d matrix states (density kind): column-major, like Eigen's MatrixXcd
        if a.ndim == 2:
            a = np.broadcast_to(a[None], (B,) + a.shape)
        if a.shape != (B, d, d):
            raise InvalidArgument(f"{what} state has shape {a.shape}, expected ({B}, {d}, {d})")
        return np.ascontiguousarray(np.swapaxes(a, 1, 2)).reshape(B, d * d)
    if a.ndim == 2 and a.shape[1] == 1 and B == 1 and a.shape[0] == d:
        a = a[:, 0]
    if a.ndim == 1:
        a = np.broadcast_to(a[None], (B, a.shape[0]))
    if a.shape != (B, d):
        raise InvalidArgument(f"{what} state has shape {a.shape}, expected ({B}, {d})")
    return np.ascontiguousarray(a)


def pack_problem(p: ControlProblem) -> abi.PackedProblem:
    if p.model is None:
        raise InvalidArgument("problem has no model")
    m = p.model
    s = abi.ProblemV1()
    keep: list = []
    s.abi_version = abi.QOC_ABI_VERSION
    s.kind = m.kind
    s.dim = m.state_dim()
    s.channels = m.channels()
    s.steps = p.grid.steps
    s.batch = m.batch
    s.t_start = p.grid.t_start
    s.dt = p.grid.dt
    s.ip_weight = m.ip_weight()
    m.pack_into(s, keep)
    sq = m.kind == abi.KIND_DENSITY
    ini = abi.cplx(_states(p.initial, m.batch, s.dim, "initial", sq))
    tgt = abi.cplx(_states(p.target, m.batch, s.dim, "target", sq))
    keep += [ini, tgt]
    s.initial, s.target = abi.dptr(ini), abi.dptr(tgt)
    if p.penalty is not None:
        pen = np.ascontiguousarray(np.broadcast_to(np.asarray(p.penalty, dtype=np.float64), (p.grid.steps,)))
        keep.append(pen)
        s.penalty = abi.dptr(pen)
    return abi.PackedProblem(s, keep)


def controls_to_abi(u, B: int, Cn: int, K: int) -> np.ndarray:
    """(C, K) or (B, C, K) samples -> [B][K][C] contiguous (column-major C x K per problem)."""
    u = np.asarray(u, dtype=np.float64)
    if u.ndim == 2:
        u = np.broadcast_to(u[None], (B,) + u.shape)
    if u.shape != (B, Cn, K):
        raise InvalidArgument(f"control has shape {u.shape}, expected ({B}, {Cn}, {K}) "
                              "(initial control grid/channel count does not match the problem)")
    return np.ascontiguousarray(np.swapaxes(u, 1, 2)).reshape(-1)


def controls_from_abi(flat: np.ndarray, B: int, Cn: int, K: int) -> np.ndarray:
    return np.ascontiguousarray(np.swapaxes(flat.reshape(B, K, Cn), 1, 2))


_VARIANTS = {"interpolated": abi.VARIANT_INTERPOLATED, "split": abi.VARIANT_SPLIT}
_PLANS = {"assembled": abi.PLAN_ASSEMBLED, "direct": abi.PLAN_DIRECT}
_PARTS = {"balanced": abi.PARTITION_BALANCED, "uniform": abi.PARTITION_UNIFORM,
          "explicit": abi.PARTITION_EXPLICIT}
_SOLVERS = {"gradient": abi.SOLVER_GRADIENT, "monotonic": abi.SOLVER_MONOTONIC,
            "newton": abi.SOLVER_NEWTON}


def pack_config(cfg: IsmConfig):
    c = abi.IsmConfigV1()
    c.subintervals, c.workers, c.max_outer = cfg.subintervals, cfg.workers, cfg.max_outer
    try:
        c.variant, c.plan = _VARIANTS[cfg.variant], _PLANS[cfg.plan]
        c.partition = _PARTS[cfg.partition]
    except KeyError as e:
        raise InvalidArgument(f"unknown option {e}") from None
    c.compute_error = int(cfg.compute_error)
    c.log_exact_objective = int(cfg.log_exact_objective)
    c.checkpoint_stride = cfg.checkpoint_stride
    c.blocks = int(cfg.blocks)
    c.eta = cfg.eta
    keep = None
    if cfg.node_index is not None:
        keep = np.ascontiguousarray(cfg.node_index, dtype=np.int32)
        c.node_index = abi.iptr(keep)
        c.partition = abi.PARTITION_EXPLICIT
    return c, keep


def pack_solver(sv: SolverSpec):
    s = abi.SolverV1()
    if sv.kind not in _SOLVERS:
        raise InvalidArgument(f"unknown solver {sv.kind}")
    s.kind = _SOLVERS[sv.kind]
    s.inner_iterations = sv.inner_iterations
    s.naive_nonlinear_adjoint = int(sv.naive_nonlinear_adjoint)
    s.checkpoint_stride = sv.checkpoint_stride
    s.step_size = sv.step_size
    s.fixed_point_tol, s.fixed_point_max_iter = sv.fixed_point_tol, sv.fixed_point_max_iter
    s.gmres_restart, s.gmres_max_iter = sv.gmres_restart, sv.gmres_max_iter
    s.gmres_tol, s.hvp_scale = sv.gmres_tol, sv.hvp_scale
    return s


def unpack_records(recs: np.ndarray, tvals: np.ndarray, status, cfg: IsmConfig,
                   solver: SolverSpec, b: int) -> RunRecord:
    return unpack_all(recs[b:b + 1], tvals[b:b + 1], [status[b]], cfg, solver)[0]


def solver_events(stats_row) -> list:
    """The per-task inner-solver events of one iteration (ism.cpp:503-511) from its counters
    stats_row[3][L] = guard_rejections, newton_fallbacks, gmres_iterations."""
    ev = []
    for n in range(stats_row.shape[1]):
        if stats_row[0, n] > 0:
            ev.append(f"task {n}: kept {int(stats_row[0, n])} slices at previous values")
        if stats_row[1, n] > 0:
            ev.append(f"task {n}: {int(stats_row[1, n])} Newton directions replaced by gradient steps")
    return ev


def unpack_all(recs: np.ndarray, tvals: np.ndarray, status, cfg: IsmConfig, solver: SolverSpec,
               task_value_lists: bool = True, stats=None) -> list:
    """RunRecords of every batch member.  With task_value_lists=False each IterationStat.task_values
    is a read-only row view of `tvals`; the IterationStat objects are built lazily per record.
    stats(b, k) -> int array [3][L] of the inner-solver counters (or None)."""
    if not task_value_lists:
        tvals.setflags(write=False)

    def builder(b: int, n: int, aborted: bool, reason: str):
        def build():
            rb = recs[b, :n]
            it_, obj, ex = rb["iteration"].tolist(), rb["objective"].tolist(), rb["exact_objective"].tolist()
            er, sec = rb["error"].tolist(), rb["device_seconds"].tolist()
            hx, he = rb["has_exact_objective"].tolist(), rb["has_error"].tolist()
            tv = tvals[b, :n].tolist() if task_value_lists else tvals[b]
            its = [IterationStat(iteration=it_[k], objective=obj[k], exact_objective=ex[k] if hx[k] else None,
                                 error=er[k] if he[k] else None, task_values=tv[k], device_seconds=sec[k])
                   for k in range(n)]
            if stats is not None:
                for k in range(1, n):
                    row = stats(b, k)
                    if row is not None:
                        its[k].solver_stats = row
                        its[k].events.extend(solver_events(row))
            if aborted and its:  # the stopping iteration carries the reason
                its[-1].events.append(reason)
            return its
        return build

    out = []
    for b, st in enumerate(status):
        rec = RunRecord(subintervals=cfg.subintervals, workers=cfg.workers, solver=solver.kind,
                        variant=cfg.variant, plan=cfg.plan, aborted=bool(st.aborted),
                        abort_reason=st.abort_reason.decode())
        rec._build = builder(b, st.iterations_recorded, rec.aborted, rec.abort_reason)
        out.append(rec)
    return out


def run_buffers(p: ControlProblem, cfg: IsmConfig):
    B, L = p.batch, cfg.subintervals
    cap = max(cfg.max_outer, 0) + 1
    recs = np.zeros((B, cap), dtype=abi.REC_DTYPE)
    tvals = np.empty((B, cap, max(L, 1)))  # every entry is written by the device (NaN where unset)
    status = (abi.RunStatusV1 * B)()
    return cap, recs, tvals, status


def _validate(p: ControlProblem, cfg: IsmConfig) -> None:
    if cfg.variant == "interpolated" and not p.model.is_linear():
        raise InvalidArgument("interpolated waypoints require linear one-step flows; use the split "
                              "variant for split-step states")


# ----------------------------------------------------------------------------------------
# The device entry points.
# ----------------------------------------------------------------------------------------
def run_ism_batch(p: ControlProblem, u0, cfg: IsmConfig, solver: SolverSpec,
                  ctx=None) -> list[IsmRun]:
    """run_ism for every problem of a batched ControlProblem, in one device call."""
    from . import _native
    _validate(p, cfg)
    packed = pack_problem(p)
    B, Cn, K = p.batch, p.model.channels(), p.grid.steps
    u_in = controls_to_abi(u0, B, Cn, K)
    u_out = np.empty_like(u_in)
    c, keep = pack_config(cfg)
    s = pack_solver(solver)
    cap, recs, tvals, status = run_buffers(p, cfg)
    ctx = ctx or _native.default_context()
    code = ctx.lib.qoc_ism_run(ctx.handle, packed.ref, C.byref(c), C.byref(s), abi.dptr(u_in),
                               abi.dptr(u_out), recs.ctypes.data_as(C.c_void_p), cap,
                               abi.dptr(tvals), status)
    raise_for(code, ctx.last_error())
    u = controls_from_abi(u_out, B, Cn, K)
    stats = None
    if solver.kind != "gradient":
        L = cfg.subintervals

        def stats(b, k, _ctx=ctx):
            row = np.zeros((3, L), dtype=np.int32)
            ok = _ctx.lib.qoc_ctx_solver_stats(_ctx.handle, b, k, L, row.ctypes.data_as(C.c_void_p))
            return row if ok == abi.QOC_OK else None
    return [IsmRun(u[b], r) for b, r in enumerate(unpack_all(recs, tvals, status, cfg, solver, B == 1, stats))]


def run_ism(p: ControlProblem, u0, cfg: IsmConfig, solver: SolverSpec, ctx=None) -> IsmRun:
    """ism.hpp:80-81 -- single-problem solve on the device."""
    if p.batch != 1:
        raise InvalidArgument("run_ism takes one problem; use run_ism_batch")
    return run_ism_batch(p, u0, cfg, solver, ctx)[0]


def state_shape(model) -> tuple:
    """Shape of one state: (d,) vectors, or (d, d) matrices for the density kind."""
    d = model.state_dim()
    return (d, d) if model.kind == abi.KIND_DENSITY else (d,)


def unpack_states(flat: np.ndarray, model, lead: tuple) -> np.ndarray:
    """Interleaved complex states (column-major matrices for the density kind) -> numpy."""
    z = flat.view(np.complex128)
    shp = state_shape(model)
    if len(shp) == 2:
        return np.swapaxes(z.reshape(lead + (shp[1], shp[0])), -1, -2)
    return z.reshape(lead + shp)


def imaginary_time(model, u_frozen, psi0, imaginary_dt: float = 1e-2, energy_tol: float = 1e-10,
                   max_iterations: int = 200000, lower=None, ctx=None):
    """Stationary states of a condensate model by normalized imaginary-time splitting on the
    device (the first stage of ground_state, models.cpp:129-182), one CTA per frozen control.

    u_frozen: (S,) controls; psi0: (S, d) or (d,) starting guesses; lower: optional (S, Q, d) or
    (Q, d) states projected out every iteration (excited states).  Returns (psi (S, d),
    energy (S,), iterations (S,))."""
    from . import _native
    u = np.ascontiguousarray(np.atleast_1d(np.asarray(u_frozen, dtype=np.float64)))
    S, d = u.size, model.state_dim()
    psi = np.ascontiguousarray(np.broadcast_to(np.asarray(psi0, dtype=np.complex128), (S, d))).copy()
    grid = TimeGrid.over(0.0, 1.0, 1)
    prob = ControlProblem(model, grid, psi[0], psi[0], None)
    packed = pack_problem(prob)
    nl, low = 0, None
    if lower is not None:
        low = np.asarray(lower, dtype=np.complex128)
        if low.ndim == 2:
            low = np.broadcast_to(low, (S,) + low.shape)
        low = np.ascontiguousarray(low)
        nl = low.shape[1]
    buf = abi.cplx(psi)
    lowbuf = abi.cplx(low) if nl else None
    en, its = np.empty(S), np.empty(S, dtype=np.int32)
    ctx = ctx or _native.default_context()
    raise_for(ctx.lib.qoc_imaginary_time(ctx.handle, packed.ref, S, abi.dptr(u), float(imaginary_dt),
                                         float(energy_tol), int(max_iterations), nl,
                                         abi.dptr(lowbuf) if nl else None, abi.dptr(buf), abi.dptr(en),
                                         its.ctypes.data_as(C.c_void_p)), ctx.last_error())
    return buf.view(np.complex128).reshape(S, d), en, its


def propagate_final(p: ControlProblem, u, ctx=None) -> np.ndarray:
    """propagation.cpp:194-200, on the device: (B,) + state shape final states."""
    from . import _native
    packed = pack_problem(p)
    B, Cn, K = p.batch, p.model.channels(), p.grid.steps
    u_in = controls_to_abi(u, B, Cn, K)
    out = np.empty(2 * B * int(np.prod(state_shape(p.model))))
    ctx = ctx or _native.default_context()
    raise_for(ctx.lib.qoc_propagate_final(ctx.handle, packed.ref, abi.dptr(u_in), abi.dptr(out)),
              ctx.last_error())
    return unpack_states(out, p.model, (B,))


def objective_gradient(p: ControlProblem, u, form: str = "tracking", naive: bool = False, ctx=None):
    """evaluate_objective + objective_gradient (objective.cpp:93-129) on the device.
    Returns (values (B,), gradients (B, C, K))."""
    from . import _native
    packed = pack_problem(p)
    B, Cn, K = p.batch, p.model.channels(), p.grid.steps
    u_in = controls_to_abi(u, B, Cn, K)
    val = np.empty(B)
    grad = np.empty_like(u_in)
    f = abi.FORM_OVERLAP if form == "overlap" else abi.FORM_TRACKING
    ctx = ctx or _native.default_context()
    raise_for(ctx.lib.qoc_objective_gradient(ctx.handle, packed.ref, abi.dptr(u_in), f, int(naive),
                                             abi.dptr(val), abi.dptr(grad)), ctx.last_error())
    return val, controls_from_abi(grad, B, Cn, K)


def evaluate_objective(p: ControlProblem, u, form: str = "tracking", ctx=None) -> np.ndarray:
    from . import _native
    packed = pack_problem(p)
    B, Cn, K = p.batch, p.model.channels(), p.grid.steps
    u_in = controls_to_abi(u, B, Cn, K)
    val = np.empty(B)
    f = abi.FORM_OVERLAP if form == "overlap" else abi.FORM_TRACKING
    ctx = ctx or _native.default_context()
    raise_for(ctx.lib.qoc_objective_gradient(ctx.handle, packed.ref, abi.dptr(u_in), f, 0,
                                             abi.dptr(val), None), ctx.last_error())
    return val


def assemble_propagator(p: ControlProblem, u, ctx=None) -> np.ndarray:
    """propagation.cpp:236-249 on the device: (B, d, d) products of the one-step maps."""
    from . import _native
    packed = pack_problem(p)
    B, Cn, K, d = p.batch, p.model.channels(), p.grid.steps, p.model.state_dim()
    u_in = controls_to_abi(u, B, Cn, K)
    out = np.empty(2 * B * d * d)
    ctx = ctx or _native.default_context()
    raise_for(ctx.lib.qoc_assemble_propagator(ctx.handle, packed.ref, abi.dptr(u_in), abi.dptr(out)),
              ctx.last_error())
    return np.swapaxes(out.view(np.complex128).reshape(B, d, d), 1, 2)


def balanced_nodes(K: int, L: int) -> list[int]:
    """The balanced decomposition: first K mod L parts get ceil(K/L) steps."""
    base, extra = divmod(K, L)
    nodes = [0]
    for n in range(L):
        nodes.append(nodes[-1] + base + (1 if n < extra else 0))
    return nodes


def fidelity_history(run: IsmRun, split: bool = False) -> np.ndarray:
    """F_k per SURVEY §8(d): 1 + objective (interpolated, alpha = 0) or exact_objective."""
    its = run.record.iterations
    if split:
        return np.array([it.exact_objective if it.exact_objective is not None else math.nan for it in its])
    return np.array([1.0 + it.objective for it in its])

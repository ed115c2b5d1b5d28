"""Problem builders: the five BASELINE.json configs and the reference's condensate preset.

Setup only (host, numpy): nothing here is on the timed path.  Seeds, generator and draw
order are the ones pinned in SURVEY.md §8(d) ("Seeds and generator"): numpy PCG64
``default_rng(seed)``; complex Gaussians drawn real part then imaginary part per element,
elements in column-major order.  Unspecified BASELINE parameters are pinned as SURVEY §8(d)
proposes and echoed by :func:`describe`.

No public dataset is involved: every config is a synthetic physics problem defined by its
operators, states and seeded first-guess control.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import abi
from .ism import ControlProblem, IsmConfig, SolverSpec, TimeGrid
from .models import CondensateModel, DenseModel, DensityModel, SpinRegisterModel, TridiagonalModel

SX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
SY = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
SZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)


@dataclass
class Workload:
    name: str
    problem: ControlProblem
    u0: np.ndarray
    config: IsmConfig
    solver: SolverSpec
    rho_fast: float              # rho = 0.1/dt (time-to-fidelity runs)
    notes: dict = field(default_factory=dict)


def complex_gaussian(rng: np.random.Generator, shape) -> np.ndarray:
    """Real then imaginary part per element, elements in column-major order."""
    n = int(np.prod(shape))
    z = rng.standard_normal(2 * n)
    v = z[0::2] + 1j * z[1::2]
    return v.reshape(tuple(reversed(shape))).T if len(shape) == 2 else v.reshape(shape)


# --------------------------------------------------------------------------------------
# Config 1: two coupled spins (d = 4).
# --------------------------------------------------------------------------------------
def spin2(iterations: int = 200, rho: float = 0.1, subintervals: int = 8) -> Workload:
    J = 1.0
    h0 = (np.pi * J / 2) * np.kron(SZ, SZ)
    hc = (np.kron(SX, I2) + np.kron(I2, SX)) / 2
    K, T = 1000, 10.0
    psi_i = np.zeros(4, complex); psi_i[0] = 1.0
    psi_t = np.zeros(4, complex); psi_t[3] = 1.0
    u0 = (0.1 + 0.05 * np.random.default_rng(1).standard_normal(K)).reshape(1, K)
    grid = TimeGrid.over(0.0, T, K)
    p = ControlProblem(DenseModel(h0, [hc]), grid, psi_i, psi_t, np.zeros(K))
    cfg = IsmConfig(subintervals=subintervals, workers=8, eta=0.0, max_outer=iterations)
    return Workload("spin2", p, u0, cfg, SolverSpec(step_size=rho), 0.1 / grid.dt)


# --------------------------------------------------------------------------------------
# Config 2: linear rigid rotor, j = 0..20 (d = 21), tridiagonal.
# --------------------------------------------------------------------------------------
def rotor_coupling(j_max: int) -> np.ndarray:
    """<j|cos theta|j+1> = (j+1)/sqrt((2j+1)(2j+3))  (orientation_coupling, models.cpp:349-359)."""
    j = np.arange(j_max, dtype=np.float64)
    return (j + 1.0) / np.sqrt((2.0 * j + 1.0) * (2.0 * j + 3.0))


def rotor21(subintervals: int = 128, iterations: int = 200, rho: float = 0.1,
            tridiagonal: bool = True) -> Workload:
    j_max, B, mu = 20, 1.0, 1.0
    d = j_max + 1
    j = np.arange(d, dtype=np.float64)
    diag = np.stack([B * j * (j + 1.0), np.zeros(d)])
    sub = np.stack([np.zeros(d - 1, complex), -mu * rotor_coupling(j_max).astype(complex)])
    model = TridiagonalModel(diag, sub, channels=1)
    if not tridiagonal:
        model = model.to_dense()
    K, T = 20000, 20.0
    psi_i = np.zeros(d, complex); psi_i[0] = 1.0
    t = complex_gaussian(np.random.default_rng(2), (5,))
    psi_t = np.zeros(d, complex); psi_t[:5] = t / np.linalg.norm(t)
    u0 = np.random.default_rng(3).uniform(-0.5, 0.5, K).reshape(1, K)
    grid = TimeGrid.over(0.0, T, K)
    p = ControlProblem(model, grid, psi_i, psi_t, np.zeros(K))
    cfg = IsmConfig(subintervals=subintervals, workers=8, eta=0.0, max_outer=iterations)
    return Workload("rotor21", p, u0, cfg, SolverSpec(step_size=rho), 0.1 / grid.dt)


# --------------------------------------------------------------------------------------
# Config 3: Ising chain, n = 10 (d = 1024), bit-flip operator form.
# --------------------------------------------------------------------------------------
def ising_diag(J: np.ndarray, n: int) -> np.ndarray:
    """sum_i J_i z_i z_{i+1} (open chain), z = +1 for bit 0 (spin up); spin i = bit n-1-i."""
    s = np.arange(1 << n)
    z = np.stack([1.0 - 2.0 * ((s >> (n - 1 - i)) & 1) for i in range(n)])
    return np.sum(J[:, None] * z[:-1] * z[1:], axis=0)


def ising10(subintervals: int = 256, iterations: int = 20, rho: float = 0.1, nspins: int = 10,
            steps: int = 4000, T: float = 30.0) -> Workload:
    n = nspins
    J = np.random.default_rng(4).uniform(0.5, 1.5, n - 1)
    model = SpinRegisterModel(n, ising_diag(J, n), [0, 1], np.full((2, n), 0.5))
    d = 1 << n
    psi_i = np.zeros(d, complex); psi_i[0] = 1.0
    psi_t = np.zeros(d, complex); psi_t[-1] = 1.0
    z = np.random.default_rng(5).standard_normal(2 * steps)
    u0 = (0.1 + 0.05 * z).reshape(2, steps)  # channel x then channel y
    grid = TimeGrid.over(0.0, T, steps)
    p = ControlProblem(model, grid, psi_i, psi_t, np.zeros(steps))
    # direct plan: the spin register never forms its d x d one-step matrices (16 MB each at
    # d = 1024) on one GPU; direct and assembled agree to rounding (ism_test.cpp:248-265)
    cfg = IsmConfig(subintervals=subintervals, workers=8, eta=0.0, max_outer=iterations, plan="direct")
    return Workload("ising10", p, u0, cfg, SolverSpec(step_size=rho), 0.1 / grid.dt)


# --------------------------------------------------------------------------------------
# The reference's `spins` preset: density-matrix (conjugation) transfer on a coupled chain
# (models.cpp:320-347, config.cpp:128-146; the paper's 5-spin benchmark).
# --------------------------------------------------------------------------------------
def spin_operator(n: int, k: int, axis: str) -> np.ndarray:
    """sigma_axis / 2 on spin k of n (spin 0 = most significant factor, models.cpp:296-318)."""
    s = {"x": SX, "y": SY, "z": SZ}[axis] / 2
    op = np.eye(1, dtype=np.complex128)
    for i in range(n):
        op = np.kron(op, s if i == k else I2)
    return op


def default_couplings(n: int):  # config.cpp:79-93
    if n == 5:
        return [(1, 2), (1, 3), (2, 3), (2, 5), (3, 4)]
    if n == 3:
        return [(1, 2), (1, 3), (2, 3)]
    return [(a, a + 1) for a in range(1, n)]


def spins_preset(quick: bool = True, subintervals: int = 4, iterations=None, steps=None, seed: int = 7) -> Workload:
    """spin_chain_problem (models.cpp:320-347) with the preset parameters (config.cpp:132-146;
    SpinsParams defaults config.hpp:21-28): n = 3 (quick) or 5 spins, J = 140, duration 0.14 or
    14, 2^10 or 2^15 steps, alpha = 0, gradient rho = 1e4, interpolated variant, initial control
    uniform in [-1, 1] (the reference draws it with std::mt19937 seed 7; here numpy PCG64 seed 7)."""
    n = 3 if quick else 5
    J, T = 140.0, (0.14 if quick else 14.0)
    K = steps or (1 << 10 if quick else 1 << 15)
    h0 = sum(2.0 * np.pi * J * (spin_operator(n, a - 1, "z") @ spin_operator(n, b - 1, "z"))
             for a, b in default_couplings(n))
    ctl = []
    for k in range(n):
        ctl += [spin_operator(n, k, "x"), spin_operator(n, k, "y")]
    grid = TimeGrid.over(0.0, T, K)
    p = ControlProblem(DensityModel(h0, np.stack(ctl)), grid, spin_operator(n, 0, "x"),
                       spin_operator(n, n - 1, "x"), np.zeros(K))
    u0 = np.random.default_rng(seed).uniform(-1.0, 1.0, (2 * n, K))
    cfg = IsmConfig(subintervals=subintervals, workers=8, eta=0.0, max_outer=iterations or (25 if quick else 50))
    return Workload("spins", p, u0, cfg, SolverSpec(step_size=1e4), 0.1 / grid.dt)


# --------------------------------------------------------------------------------------
# Config 5: batch of random 4-qubit problems (d = 16).
# --------------------------------------------------------------------------------------
def batch_problems(batch: int = 4096, d: int = 16, seed_base: int = 1000, u_seed_base: int = 100000,
                   steps: int = 2000):
    h0 = np.empty((batch, d, d), complex)
    hc = np.empty((batch, d, d), complex)
    psi_i = np.empty((batch, d), complex)
    psi_t = np.empty((batch, d), complex)
    u0 = np.empty((batch, 1, steps))
    for b in range(batch):
        rng = np.random.default_rng(seed_base + b)
        g = complex_gaussian(rng, (d, d))
        h0[b] = (g + g.conj().T) / 2 / np.sqrt(d)
        g = complex_gaussian(rng, (d, d))
        hc[b] = (g + g.conj().T) / 2 / np.sqrt(d)
        v = complex_gaussian(rng, (d,)); psi_i[b] = v / np.linalg.norm(v)
        v = complex_gaussian(rng, (d,)); psi_t[b] = v / np.linalg.norm(v)
        u0[b, 0] = 0.1 + 0.05 * np.random.default_rng(u_seed_base + b).standard_normal(steps)
    return h0, hc, psi_i, psi_t, u0


def batch4096(batch: int = 4096, subintervals: int = 128, iterations: int = 200, rho: float = 0.1,
              first: int = 0) -> Workload:
    K, T, d = 2000, 10.0, 16
    h0, hc, psi_i, psi_t, u0 = batch_problems(batch, d, 1000 + first, 100000 + first, K)
    grid = TimeGrid.over(0.0, T, K)
    p = ControlProblem(DenseModel(h0, hc[:, None]), grid, psi_i, psi_t, np.zeros(K))
    cfg = IsmConfig(subintervals=subintervals, workers=8, eta=0.0, max_outer=iterations)
    return Workload("batch4096", p, u0, cfg, SolverSpec(step_size=rho), 0.1 / grid.dt,
                    {"batch": batch, "first_problem": first})


# --------------------------------------------------------------------------------------
# Condensates: stationary states (setup; restates models.cpp:129-294 with numpy linalg).
# --------------------------------------------------------------------------------------
def _udft(x):
    return np.fft.fft(x, norm="ortho")


def _uidft(x):
    return np.fft.ifft(x, norm="ortho")


def stationary_state(model: CondensateModel, u: float, excited: int = 0, lower=None,
                     imaginary_dt: float = 1e-2, energy_tol: float = 1e-10, device: bool = False,
                     ctx=None) -> np.ndarray:
    """Self-consistent stationary state number `excited` (0 = ground) at frozen control u.

    Ground state: normalized imaginary-time splitting (models.cpp:146-182; on the device with
    device=True, qoc_imaginary_time), the normalized gradient-flow polish (models.cpp:184-242),
    then damped self-consistent diagonalization at frozen density until the residual stops
    improving (models.cpp:245-262).  Excited state (BASELINE config 4 has
    no reference code; pinned here): the same SCF selecting eigenvector `excited`, started from
    imaginary time with Gram-Schmidt against `lower`.  Phase (models.cpp:265-272): the first
    component within 1e-8 of the largest magnitude is made real positive.
    """
    v = model.potential([u])
    kin = model.kinetic
    dx, n, kappa = model.dx, model.points, model.kappa
    half_kin = np.exp(-0.5 * imaginary_dt * kin)
    x = model.x
    psi = np.exp(-0.5 * x * x).astype(complex)
    if excited:
        psi = psi * x
    lower = [] if lower is None else lower

    def orth(s):
        for q in lower:
            s = s - dx * np.vdot(q, s) * q
        return s / (np.sqrt(dx) * np.linalg.norm(s))

    def energy(s):
        hat = _udft(s)
        den = np.abs(s) ** 2
        return dx * (np.sum(kin * np.abs(hat) ** 2) + np.sum(v * den) + 0.5 * kappa * np.sum(den * den))

    def apply_h(s):
        return _uidft(kin * _udft(s)) + (v + kappa * np.abs(s) ** 2) * s

    psi = orth(psi)
    e = energy(psi)
    if device:  # the imaginary-time stage on the GPU (qoc_imaginary_time), the SCF polish below on the host
        from . import ism as _ism
        out, _, _ = _ism.imaginary_time(model, [u], psi, imaginary_dt, energy_tol, 200000,
                                        lower=np.asarray(lower) if lower else None, ctx=ctx)
        psi = out[0]
    for _ in range(0 if device else 200000):
        pa = _uidft(half_kin * _udft(psi))
        pa = pa * np.exp(-imaginary_dt * (v + kappa * np.abs(pa) ** 2))
        psi = orth(_uidft(half_kin * _udft(pa)))
        e2 = energy(psi)
        done = abs(e2 - e) < energy_tol
        e = e2
        if done:
            break

    # normalized gradient flow on the exact discrete energy (models.cpp:184-242): backtracked steps
    # along -(H[psi] - mu) psi remove the O(dt^2) splitting bias of the imaginary-time fixed point
    step, e_now = imaginary_dt, energy(psi)
    for _ in range(20000):
        hs = apply_h(psi)
        r = hs - dx * np.real(np.vdot(psi, hs)) * psi
        if np.sqrt(dx) * np.linalg.norm(r) < 1e-12:
            break
        accepted = False
        for _back in range(60):
            trial = orth(psi - step * r)
            e_trial = energy(trial)
            if e_trial <= e_now + 4e-16 * (1.0 + abs(e_now)):
                psi, e_now, accepted = trial, e_trial, True
                step *= 1.25
                break
            step *= 0.5
        if not accepted:
            break  # descent stalled at the rounding floor

    eye = np.eye(n)
    kd = np.stack([_uidft(kin * _udft(eye[:, c])) for c in range(n)], axis=1)
    kd = 0.5 * (kd + kd.conj().T)
    density = np.abs(psi) ** 2

    def resid(s):
        hs = apply_h(s)
        mu = dx * np.real(np.vdot(s, hs))
        return np.sqrt(dx) * np.linalg.norm(hs - mu * s)

    best = resid(psi)
    stale = 0
    for _ in range(500):
        if best <= 1e-13:
            break
        w, vecs = np.linalg.eigh(kd + np.diag(v + kappa * density))
        cand = vecs[:, excited] / np.sqrt(dx)
        if excited and np.real(np.vdot(psi, cand)) < 0:
            cand = -cand
        r = resid(cand)
        if r < best:
            best, psi, stale = r, cand.astype(complex), 0
        else:
            stale += 1
            if stale > 25:
                break
        density = 0.5 * density + 0.5 * np.abs(psi) ** 2
    mag = np.abs(psi)
    pivot = int(np.argmax(mag >= (1.0 - 1e-8) * mag.max()))
    psi = psi * np.conj(psi[pivot]) / np.abs(psi[pivot])
    return psi


def ramp_control(grid: TimeGrid, start: float, stop: float) -> np.ndarray:
    """midpoint-sampled ramp (models.cpp:429-437)."""
    span = grid.dt * grid.steps
    j = np.arange(grid.steps)
    mid = (grid.t_start + grid.dt * j) + 0.5 * grid.dt - grid.t_start
    return (start + (stop - start) * (mid / span)).reshape(1, -1)


def condensate_preset(subintervals: int = 4, iterations: int = 10) -> Workload:
    """The reference's 'condensate' preset (config.cpp:151-165, CondensateParams config.hpp:39-47)
    as used by acceptance criterion 8 (acceptance_main.cpp:439-485, KAT-8)."""
    model = CondensateModel(50, -10.0, 10.0, abi.POT_TRAP, [10.0], 1.0)
    grid = TimeGrid.over(0.0, 8.0, 1 << 9)
    psi_i = stationary_state(model, 1.0)
    psi_t = stationary_state(model, 0.0)
    p = ControlProblem(model, grid, psi_i, psi_t, np.zeros(grid.steps))
    cfg = IsmConfig(subintervals=subintervals, workers=1, eta=0.0, max_outer=iterations,
                    variant="split", log_exact_objective=True)
    return Workload("condensate", p, ramp_control(grid, 1.0, 0.0), cfg, SolverSpec(step_size=0.1),
                    0.1 / grid.dt)


_GPE_STATES: dict = {}


def gpe1024(subintervals: int = 64, iterations: int = 100, rho: float = 0.1, points: int = 1024,
            steps: int = 10000, T: float = 5.0) -> Workload:
    """BASELINE config 4: H = -1/2 d2/dx2 + x^2/2 + 5 cos^2(x - u) + 10|psi|^2 on [-16, 16)."""
    model = CondensateModel(points, -16.0, 16.0, abi.POT_LATTICE, [1.0, 5.0, 1.0], 10.0)
    if points not in _GPE_STATES:  # setup only; memoised per process (~20 s at 1024 points)
        g = stationary_state(model, 0.0)
        _GPE_STATES[points] = (g, stationary_state(model, 0.0, excited=1, lower=[g]))
    psi_i, psi_t = (s.copy() for s in _GPE_STATES[points])
    grid = TimeGrid.over(0.0, T, steps)
    p = ControlProblem(model, grid, psi_i, psi_t, np.zeros(steps))
    cfg = IsmConfig(subintervals=subintervals, workers=8, eta=0.0, max_outer=iterations,
                    variant="split", log_exact_objective=True)
    return Workload("gpe1024", p, np.zeros((1, steps)), cfg, SolverSpec(step_size=rho), 0.1 / grid.dt)


BUILDERS = {"spin2": spin2, "rotor21": rotor21, "ising10": ising10, "gpe1024": gpe1024,
            "batch4096": batch4096, "condensate": condensate_preset}


def describe(w: Workload) -> dict:
    from .ism import balanced_nodes
    p, c = w.problem, w.config
    nodes = balanced_nodes(p.grid.steps, c.subintervals)
    lens = np.diff(nodes)
    part = {int(n): int(np.sum(lens == n)) for n in np.unique(lens)}
    return {"workload": w.name, "dim": p.model.state_dim(), "channels": p.model.channels(),
            "steps": p.grid.steps, "dt": p.grid.dt, "subintervals": c.subintervals,
            "partition": " + ".join(f"{v}x{k}" for k, v in sorted(part.items(), reverse=True)),
            "batch": p.batch, "variant": c.variant, "plan": c.plan,
            "step_size": w.solver.step_size, **w.notes}

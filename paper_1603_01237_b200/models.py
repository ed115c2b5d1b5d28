"""Model plugins: the Python mirror of the reference's ``HamiltonianModel`` contract.

Reference interface: ``class HamiltonianModel`` (propagation.hpp:20-38) with the concrete
``DenseModel`` (models.hpp:15-31, models.cpp:45-75) and ``TrappedCondensateModel``
(models.hpp:40-64, models.cpp:77-127).  Each class here carries the operator payload of one
``qoc_kind`` of ``include/qoc_gpu.h`` and packs it into ``qoc_problem_v1``.  Every operator
array may carry a leading batch axis B (independent problems sharing d, C and the grid).

Operators are plain numpy arrays (row-major ``[i, j]`` indexing); packing converts them to
the column-major complex layout of the ABI.
"""
from __future__ import annotations

import numpy as np

from . import abi


def _batched(a, ndim_single: int, dtype) -> np.ndarray:
    a = np.asarray(a, dtype=dtype)
    if a.ndim == ndim_single:
        a = a[None]
    if a.ndim != ndim_single + 1:
        raise ValueError(f"expected {ndim_single} or {ndim_single + 1} dims, got shape {a.shape}")
    return a


def _hermiticity_defect(m: np.ndarray) -> float:
    return float(np.max(np.abs(m - np.conj(np.swapaxes(m, -1, -2))))) if m.size else 0.0


class HamiltonianModel:
    """Base of the plugin classes (propagation.hpp:20-38)."""

    kind: int = -1
    batch: int = 1

    def state_dim(self) -> int:
        raise NotImplementedError

    def channels(self) -> int:
        raise NotImplementedError

    def ip_weight(self) -> float:
        return 1.0

    def is_linear(self) -> bool:
        return self.kind != abi.KIND_STRANG

    def pack_into(self, s: abi.ProblemV1, keep: list) -> None:
        raise NotImplementedError


class DenseModel(HamiltonianModel):
    """H(u) = H0 + sum_c u_c A_c + sum_c (u_c^2/2) B_c  (models.hpp:12-31)."""

    kind = abi.KIND_DENSE

    def __init__(self, h0, linear, quadratic=None):
        self.h0 = _batched(h0, 2, np.complex128)
        self.batch, d, d2 = self.h0.shape
        if d != d2 or d < 1:
            raise ValueError("free Hamiltonian must be square")
        lin = np.asarray(linear, dtype=np.complex128)
        if lin.ndim == 3:
            lin = np.broadcast_to(lin[None], (self.batch,) + lin.shape)
        if lin.ndim != 4 or lin.shape[0] != self.batch or lin.shape[2:] != (d, d) or lin.shape[1] < 1:
            raise ValueError("control operator dimension mismatch")
        self.linear = np.ascontiguousarray(lin)
        self.quadratic = None
        if quadratic is not None and len(quadratic):
            q = np.asarray(quadratic, dtype=np.complex128)
            if q.ndim == 3:
                q = np.broadcast_to(q[None], (self.batch,) + q.shape)
            if q.shape != self.linear.shape:
                raise ValueError("quadratic terms must be absent or given per channel")
            self.quadratic = np.ascontiguousarray(q)
        for m, what in ((self.h0, "free Hamiltonian"), (self.linear, "control operator"),
                        (self.quadratic, "quadratic operator")):
            if m is not None:
                scale = max(1.0, float(np.max(np.abs(m))))
                if _hermiticity_defect(m) > 1e-10 * scale:
                    raise ValueError(f"{what} must be Hermitian")

    def state_dim(self):
        return self.h0.shape[-1]

    def channels(self):
        return self.linear.shape[1]

    def hamiltonian(self, u, b: int = 0) -> np.ndarray:  # models.cpp:57-68
        u = np.asarray(u, dtype=np.float64)
        h = self.h0[b].copy()
        for c in range(self.channels()):
            h += u[c] * self.linear[b, c]
        if self.quadratic is not None:
            for c in range(self.channels()):
                h += (0.5 * u[c] * u[c]) * self.quadratic[b, c]
        return h

    def pack_into(self, s, keep):
        h0 = abi.cplx(abi.colmajor(self.h0))
        lin = abi.cplx(abi.colmajor(self.linear))
        keep += [h0, lin]
        s.h0, s.linear = abi.dptr(h0), abi.dptr(lin)
        if self.quadratic is not None:
            q = abi.cplx(abi.colmajor(self.quadratic))
            keep.append(q)
            s.quadratic = abi.dptr(q)


class DensityModel(DenseModel):
    """DenseModel with PropagatorKind::cn_conjugation (propagation.cpp:92-129): the states are
    d x d matrices stepped rho' = A rho A^dag (the reference's `spins` preset, models.cpp:320-347).
    state_dim() is the edge size d (propagation.hpp:25); the packed states are d*d long."""

    kind = abi.KIND_DENSITY

    def state_len(self) -> int:
        return self.state_dim() ** 2


class TridiagonalModel(HamiltonianModel):
    """DenseModel whose H0, A_c (and B_c) are Hermitian tridiagonal (rotor, models.cpp:349-359).

    ``diag[..., op, j]`` real, ``sub[..., op, j]`` = entry (j+1, j); op order H0, A_c.., B_c..
    """

    kind = abi.KIND_TRIDIAG

    def __init__(self, diag, sub, channels: int, quadratic: bool = False):
        self.diag = _batched(diag, 2, np.float64)
        self.sub = _batched(sub, 2, np.complex128)
        self.batch, nops, d = self.diag.shape
        self.C = channels
        self.has_quadratic = bool(quadratic)
        if nops != 1 + channels * (2 if quadratic else 1):
            raise ValueError("operator count does not match the channel count")
        if self.sub.shape != (self.batch, nops, d - 1):
            raise ValueError("sub-diagonal shape mismatch")

    @classmethod
    def from_dense(cls, model: DenseModel) -> "TridiagonalModel":
        ops = [model.h0[:, None]] + [model.linear]
        if model.quadratic is not None:
            ops.append(model.quadratic)
        full = np.concatenate(ops, axis=1)  # (B, nops, d, d)
        d = full.shape[-1]
        band = np.abs(np.subtract.outer(np.arange(d), np.arange(d))) > 1
        if np.any(full[..., band] != 0):
            raise ValueError("operators are not tridiagonal")
        diag = np.real(np.diagonal(full, axis1=-2, axis2=-1))
        sub = np.diagonal(full, offset=-1, axis1=-2, axis2=-1)
        return cls(diag, sub, model.channels(), model.quadratic is not None)

    def to_dense(self) -> DenseModel:
        d = self.state_dim()
        full = np.zeros(self.diag.shape[:2] + (d, d), dtype=np.complex128)
        idx = np.arange(d)
        full[..., idx, idx] = self.diag
        full[..., idx[1:], idx[:-1]] = self.sub
        full[..., idx[:-1], idx[1:]] = np.conj(self.sub)
        C = self.C
        return DenseModel(full[:, 0], full[:, 1:1 + C], full[:, 1 + C:] if self.has_quadratic else None)

    def state_dim(self):
        return self.diag.shape[-1]

    def channels(self):
        return self.C

    def pack_into(self, s, keep):
        dg = np.ascontiguousarray(self.diag, dtype=np.float64).reshape(-1)
        sb = abi.cplx(self.sub)
        keep += [dg, sb]
        s.tri_diag, s.tri_sub = abi.dptr(dg), abi.dptr(sb)
        s.tri_has_quadratic = int(self.has_quadratic)


class SpinRegisterModel(HamiltonianModel):
    """n spin-1/2 register: H(u) = diag(h0) + sum_c u_c sum_i coef[c, i] sigma^{axis_c}_i.

    Pauli matrices; spin i <-> bit (n-1-i) of the basis index (spin 0 most significant,
    the kron order of ``spin_operator``, models.cpp:296-318); |up> = bit 0.
    """

    kind = abi.KIND_BITFLIP

    def __init__(self, nspins: int, h0_diag, axes, coef):
        self.nspins = int(nspins)
        self.h0_diag = _batched(h0_diag, 1, np.float64)
        self.batch, d = self.h0_diag.shape
        if d != 1 << self.nspins:
            raise ValueError("bit-flip dim must be 2^nspins")
        self.axes = np.asarray(axes, dtype=np.int32).reshape(-1)
        self.coef = _batched(coef, 2, np.float64)
        if self.coef.shape != (self.batch, len(self.axes), self.nspins):
            raise ValueError("coefficient shape must be (B, C, nspins)")

    def state_dim(self):
        return 1 << self.nspins

    def channels(self):
        return len(self.axes)

    def channel_matrix(self, c: int, b: int = 0) -> np.ndarray:
        d, n = self.state_dim(), self.nspins
        m = np.zeros((d, d), dtype=np.complex128)
        s = np.arange(d)
        for i in range(n):
            mask = 1 << (n - 1 - i)
            g = self.coef[b, c, i]
            if self.axes[c] == 0:
                m[s, s ^ mask] += g
            else:
                one = (s & mask) != 0  # (sigma_y psi)_s = (+i if bit set else -i) psi_{s^mask}
                m[s, s ^ mask] += g * np.where(one, 1j, -1j)
        return m

    def to_dense(self) -> DenseModel:
        B, Cn = self.batch, self.channels()
        h0 = np.zeros((B, self.state_dim(), self.state_dim()), dtype=np.complex128)
        idx = np.arange(self.state_dim())
        h0[:, idx, idx] = self.h0_diag
        lin = np.stack([np.stack([self.channel_matrix(c, b) for c in range(Cn)]) for b in range(B)])
        return DenseModel(h0, lin)

    def pack_into(self, s, keep):
        dg = np.ascontiguousarray(self.h0_diag).reshape(-1)
        ax = np.ascontiguousarray(self.axes, dtype=np.int32)
        cf = np.ascontiguousarray(self.coef).reshape(-1)
        keep += [dg, ax, cf]
        s.h0, s.bf_axis, s.bf_coef = abi.dptr(dg), abi.iptr(ax), abi.dptr(cf)
        s.nspins = self.nspins


class CondensateModel(HamiltonianModel):
    """Periodic-grid condensate, split-step propagation (TrappedCondensateModel,
    models.hpp:33-64, models.cpp:77-127), with either the reference's trap potential or the
    cos^2 lattice of BASELINE config 4."""

    kind = abi.KIND_STRANG

    def __init__(self, points: int, x_min: float, x_max: float, potential: int, params, kappa: float):
        if points < 2:
            raise ValueError("grid needs at least two points")
        if not x_max > x_min:
            raise ValueError("empty space domain")
        length = x_max - x_min
        self.dx = length / points
        i = np.arange(points)
        self.x = x_min + i * self.dx  # x_min + i*dx, models.cpp:84-86
        folded = np.where(i <= points // 2, i, i - points)
        k = 2.0 * np.pi * folded / length
        self.kinetic = 0.5 * k * k
        self.potential_kind = int(potential)
        self.params = np.zeros(4)
        self.params[: len(params)] = params
        self.kappa = float(kappa)
        self.x_min, self.x_max, self.points = x_min, x_max, points

    def state_dim(self):
        return self.points

    def channels(self):
        return 1

    def ip_weight(self):
        return self.dx

    def potential(self, u) -> np.ndarray:
        u0 = float(np.asarray(u).reshape(-1)[0])
        if self.potential_kind == abi.POT_TRAP:  # models.cpp:95-110
            ld = u0 * self.params[0]
            ax = np.abs(self.x)
            r = ax - 0.5 * ld
            return np.where(ax > 0.25 * ld, 0.5 * r * r, 0.5 * (0.125 * ld * ld - self.x * self.x))
        w2, v0, kk = self.params[:3]
        return 0.5 * w2 * self.x ** 2 + v0 * np.cos(kk * (self.x - u0)) ** 2

    def pack_into(self, s, keep):
        kin = np.ascontiguousarray(self.kinetic, dtype=np.float64)
        xs = np.ascontiguousarray(self.x, dtype=np.float64)
        keep += [kin, xs]
        s.kinetic, s.grid_x = abi.dptr(kin), abi.dptr(xs)
        s.potential = self.potential_kind
        for i in range(4):
            s.pot_params[i] = float(self.params[i])
        s.kappa = self.kappa


class BasisCondensateModel(CondensateModel):
    """A condensate whose potential is supplied by the caller -- the device side of the
    reference's virtual potential(u) / potential_derivative(c, u) (propagation.hpp:35-36) -- in
    the separable form V(x_i, u) = sum_m a_m[i] f_m(u) with f_m in {u^k, cos(w u), sin(w u)}.

    terms: list of (profile a_m sampled on the grid, kind "power" | "cos" | "sin", parameter)."""

    _KINDS = {"power": abi.TERM_POWER, "cos": abi.TERM_COS, "sin": abi.TERM_SIN}

    def __init__(self, points: int, x_min: float, x_max: float, terms, kappa: float):
        super().__init__(points, x_min, x_max, abi.POT_BASIS, (), kappa)
        if not 1 <= len(terms) <= abi.MAX_POT_TERMS:
            raise ValueError(f"1..{abi.MAX_POT_TERMS} potential terms")
        self.basis = np.ascontiguousarray([np.broadcast_to(np.asarray(a, dtype=np.float64), (points,))
                                           for a, _, _ in terms])
        self.term_type = np.array([self._KINDS[k] for _, k, _ in terms], dtype=np.int32)
        self.term_param = np.array([float(q) for _, _, q in terms])
        for t, q in zip(self.term_type, self.term_param):
            if t == abi.TERM_POWER and (q < 0 or q != int(q)):
                raise ValueError("power terms take a non-negative integer exponent")

    @classmethod
    def lattice(cls, points, x_min, x_max, w2, v0, k, kappa):
        """The cos^2 lattice of BASELINE config 4 in basis form:
        v0 cos^2(k(x - u)) = v0/2 + v0/2 [cos(2kx) cos(2ku) + sin(2kx) sin(2ku)]."""
        x = x_min + np.arange(points) * ((x_max - x_min) / points)
        return cls(points, x_min, x_max, [(0.5 * w2 * x * x + 0.5 * v0, "power", 0),
                                          (0.5 * v0 * np.cos(2 * k * x), "cos", 2 * k),
                                          (0.5 * v0 * np.sin(2 * k * x), "sin", 2 * k)], kappa)

    def _f(self, u0: float, deriv: bool) -> np.ndarray:
        out = np.empty(len(self.term_type))
        for m, (t, q) in enumerate(zip(self.term_type, self.term_param)):
            if t == abi.TERM_POWER:
                k = int(q)
                out[m] = (k * u0 ** (k - 1) if k > 0 else 0.0) if deriv else u0 ** k
            elif t == abi.TERM_COS:
                out[m] = -q * np.sin(q * u0) if deriv else np.cos(q * u0)
            else:
                out[m] = q * np.cos(q * u0) if deriv else np.sin(q * u0)
        return out

    def potential(self, u) -> np.ndarray:
        return self._f(float(np.asarray(u).reshape(-1)[0]), False) @ self.basis

    def potential_derivative(self, c, u) -> np.ndarray:
        return self._f(float(np.asarray(u).reshape(-1)[0]), True) @ self.basis

    def pack_into(self, s, keep):
        super().pack_into(s, keep)
        keep += [self.basis, self.term_type, self.term_param]
        s.pot_terms = len(self.term_type)
        s.pot_term_type = abi.iptr(self.term_type)
        s.pot_term_param = abi.dptr(self.term_param)
        s.pot_basis = abi.dptr(self.basis)

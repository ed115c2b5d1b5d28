"""Loader of libqoc_b200.so (the sm_100a kernels + C-ABI host driver).

There is no fallback: if the library is missing or no B200 is visible the import of the
device path fails loudly.  Build with ``python -m paper_1603_01237_b200.build`` (or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from . import abi

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libqoc_b200.so"

_lib = None
_ctx = {}


class NativeMissing(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeMissing(f"{LIB_PATH} is not built; run `python -m paper_1603_01237_b200.build` "
                                "(the ISM path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        vp, i32, dp = C.c_void_p, C.c_int32, C.POINTER(C.c_double)
        L.qoc_abi_version.restype = i32
        L.qoc_ctx_create.argtypes = [C.POINTER(abi.CtxOptsV1), C.POINTER(vp)]
        L.qoc_ctx_create.restype = i32
        L.qoc_ctx_destroy.argtypes = [vp]
        L.qoc_ctx_destroy.restype = None
        L.qoc_ctx_last_error.argtypes = [vp]
        L.qoc_ctx_last_error.restype = C.c_char_p
        L.qoc_ctx_launch_count.argtypes = [vp]
        L.qoc_ctx_launch_count.restype = C.c_int64
        L.qoc_ctx_set_option.argtypes = [vp, i32, C.c_int64]
        L.qoc_ctx_set_option.restype = i32
        L.qoc_ctx_profile.argtypes = [vp, C.POINTER(abi.ProfileV1), i32]
        L.qoc_ctx_profile.restype = i32
        L.qoc_ctx_kernel_profile.argtypes = [vp, i32, C.c_char_p, C.c_size_t, dp, C.POINTER(C.c_int64)]
        L.qoc_ctx_kernel_profile.restype = i32
        L.qoc_ism_run.argtypes = [vp, vp, vp, vp, dp, dp, vp, i32, dp, vp]
        L.qoc_ism_run.restype = i32
        L.qoc_ctx_solver_stats.argtypes = [vp, i32, i32, i32, vp]
        L.qoc_ctx_solver_stats.restype = i32
        L.qoc_imaginary_time.argtypes = [vp, vp, i32, dp, C.c_double, C.c_double, i32, i32, dp, dp, dp, vp]
        L.qoc_imaginary_time.restype = i32
        L.qoc_propagate_final.argtypes = [vp, vp, dp, dp]
        L.qoc_propagate_final.restype = i32
        L.qoc_objective_gradient.argtypes = [vp, vp, dp, i32, i32, dp, dp]
        L.qoc_objective_gradient.restype = i32
        L.qoc_assemble_propagator.argtypes = [vp, vp, dp, dp]
        L.qoc_assemble_propagator.restype = i32
        L.qoc_comm_unique_id.argtypes = [vp, C.c_size_t]
        L.qoc_comm_unique_id.restype = i32
        L.qoc_ctx_init_comm.argtypes = [vp, i32, i32, vp, C.c_size_t]
        L.qoc_ctx_init_comm.restype = i32
        if L.qoc_abi_version() != abi.QOC_ABI_VERSION:
            raise NativeMissing("libqoc_b200.so ABI version mismatch; rebuild")
        _lib = L
    return _lib


class Context:
    """A qoc_ctx bound to one CUDA device (not thread-safe, like the C context)."""

    def __init__(self, device: int = -1):
        self.lib = lib()
        opts = abi.CtxOptsV1()
        opts.abi_version = abi.QOC_ABI_VERSION
        opts.device = device
        h = C.c_void_p()
        code = self.lib.qoc_ctx_create(C.byref(opts), C.byref(h))
        if code != abi.QOC_OK:
            raise RuntimeError(f"qoc_ctx_create failed ({code}): no sm_100 device visible?")
        self.handle = h

    def last_error(self) -> str:
        return (self.lib.qoc_ctx_last_error(self.handle) or b"").decode()

    def launches(self) -> int:
        return int(self.lib.qoc_ctx_launch_count(self.handle))

    def set_option(self, option: int, value: int) -> None:
        if self.lib.qoc_ctx_set_option(self.handle, option, int(value)) != abi.QOC_OK:
            raise RuntimeError(f"qoc_ctx_set_option({option}, {value}) failed")

    def profile(self, reset: bool = False) -> dict:
        p = abi.ProfileV1()
        self.lib.qoc_ctx_profile(self.handle, C.byref(p), int(reset))
        return {f: getattr(p, f) for f, _ in abi.ProfileV1._fields_}

    def kernel_profile(self) -> dict:
        """label -> (ms, launches) of the profiled launches since the last profile reset."""
        out, i = {}, 0
        name = C.create_string_buffer(64)
        ms, n = C.c_double(), C.c_int64()
        while self.lib.qoc_ctx_kernel_profile(self.handle, i, name, 64, C.byref(ms), C.byref(n)) == abi.QOC_OK:
            out[name.value.decode()] = (ms.value, n.value)
            i += 1
        return out

    def init_comm(self, rank: int, world: int, unique_id: bytes | None = None) -> None:
        """Bind this context to rank `rank` of a `world`-GPU NCCL communicator (qoc_ctx_init_comm);
        `unique_id` is rank 0's ``comm_unique_id()`` broadcast to every rank."""
        buf = C.create_string_buffer(bytes(unique_id), abi.COMM_ID_BYTES) if unique_id else None
        code = self.lib.qoc_ctx_init_comm(self.handle, int(rank), int(world), buf,
                                          abi.COMM_ID_BYTES if buf is not None else 0)
        if code != abi.QOC_OK:
            raise RuntimeError(f"qoc_ctx_init_comm failed ({code}): {self.last_error()}")

    def close(self):
        if self.handle:
            self.lib.qoc_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 draws it; the host side broadcasts it)."""
    buf = C.create_string_buffer(abi.COMM_ID_BYTES)
    code = lib().qoc_comm_unique_id(buf, abi.COMM_ID_BYTES)
    if code != abi.QOC_OK:
        raise RuntimeError(f"qoc_comm_unique_id failed ({code}): NCCL unavailable")
    return buf.raw


def default_context(device: int = -1) -> Context:
    if device not in _ctx:
        _ctx[device] = Context(device)
    return _ctx[device]

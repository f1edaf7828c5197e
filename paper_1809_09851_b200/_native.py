"""ctypes binding of libfvb.so (include/fvb.h).

Loading fails loudly: if the shared library is missing or cannot be loaded
the import-time helpers raise, so no code path can silently fall back to a
CPU implementation.  Status codes map to exception classes named after the
reference's error hierarchy (proj/include/fusevec/error.hpp:8-54).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_NAME = "libfvb.so"

# Symbols include/fvb.h declares; tests check the library exports each one.
EXPORTED = (
    "fvb_abi_version",
    "fvb_last_error",
    "fvb_build_info",
    "fvb_axpy_sin",
    "fvb_flux",
    "fvb_flux_prim",
    "fvb_cons2prim",
    "fvb_prim2cons",
    "fvb_v_mag2",
    "fvb_eos",
    "fvb_jacobian",
    "fvb_wave_speed_max",
    "fvb_csr_matvec_acc",
    "fvb_csr_matvec_acc_u32",
    "fvb_synth_state",
    "fvb_synth_uniform",
    "fvb_lookup",
    "fvb_emit_source",
    "fvb_nvrtc_compile",
    "fvb_pattern_count",
    "fvb_pattern",
    "fvb_ctx_create",
    "fvb_ctx_destroy",
    "fvb_flux_host",
    "fvb_jacobian_host",
    "fvb_launch_host",
)

FVB_OK = 0
FVB_ELEN = 1
FVB_EPREC = 2
FVB_ECUDA = 3
FVB_ENCCL = 4
FVB_EARG = 5
FVB_EUNSUPPORTED = 6
FVB_EALIGN = 7
FVB_EHOST = 8


class FvbError(RuntimeError):
    """Base class, the analog of fusevec::Error."""

    def __init__(self, status: int, message: str):
        super().__init__(f"[fvb status {status}] {message}")
        self.status = status


class LengthMismatch(FvbError):
    pass


class PrecisionError(FvbError):
    pass


class DeviceError(FvbError):
    pass


class ArgumentError(FvbError):
    pass


class UnsupportedExpression(FvbError):
    pass


_ERRORS = {
    FVB_ELEN: LengthMismatch,
    FVB_EPREC: PrecisionError,
    FVB_ECUDA: DeviceError,
    FVB_ENCCL: DeviceError,
    FVB_EARG: ArgumentError,
    FVB_EUNSUPPORTED: UnsupportedExpression,
    FVB_EALIGN: ArgumentError,
    FVB_EHOST: FvbError,
}


class GasStruct(ctypes.Structure):
    _fields_ = [("gamma_minus_one", ctypes.c_double), ("gamma", ctypes.c_double),
                ("cv", ctypes.c_double)]


class KernelStruct(ctypes.Structure):
    pass


KERNEL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(KernelStruct), ctypes.c_uint64,
                             ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p)

KERNEL_REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(KernelStruct), ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.c_void_p, ctypes.c_void_p)

KernelStruct._fields_ = [
    ("fn", KERNEL_FN),
    ("reduce", KERNEL_REDUCE_FN),
    ("n_outputs", ctypes.c_uint32),
    ("n_inputs", ctypes.c_uint32),
    ("n_consts", ctypes.c_uint32),
    ("prec", ctypes.c_uint8),
    ("dim", ctypes.c_uint8),
    ("in_slot", ctypes.c_int8 * 8),
    ("consts", ctypes.c_double * 8),
    ("name", ctypes.c_char * 48),
    ("impl", ctypes.c_void_p),
]


def lib_path() -> str:
    return os.environ.get("FVB_LIB", os.path.join(_HERE, "lib", _LIB_NAME))


_lock = threading.Lock()
_lib = None


def _declare(L):
    vp, u8, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint8, ctypes.c_uint32, ctypes.c_uint64, \
        ctypes.c_int
    pp = ctypes.POINTER(ctypes.c_void_p)
    gas = ctypes.POINTER(GasStruct)
    sig = {
        "fvb_abi_version": (i32, []),
        "fvb_last_error": (ctypes.c_char_p, []),
        "fvb_build_info": (ctypes.c_char_p, []),
        "fvb_axpy_sin": (i32, [u8, u64, vp, vp, vp]),
        "fvb_flux": (i32, [gas, u32, u8, u64, pp, pp, vp]),
        "fvb_flux_prim": (i32, [gas, u32, u8, u64, pp, pp, vp]),
        "fvb_cons2prim": (i32, [gas, u32, u8, u64, pp, pp, vp]),
        "fvb_prim2cons": (i32, [gas, u32, u8, u64, pp, pp, vp]),
        "fvb_v_mag2": (i32, [u32, u8, u64, pp, vp, vp]),
        "fvb_eos": (i32, [gas, u8, u64, vp, vp, vp, vp, vp]),
        "fvb_jacobian": (i32, [gas, u32, u8, u64, pp, pp, vp, vp]),
        "fvb_wave_speed_max": (i32, [gas, u32, u8, u64, pp, vp, vp, vp]),
        "fvb_csr_matvec_acc": (i32, [u8, u8, u64, u64, vp, vp, vp, vp, vp, vp]),
        "fvb_csr_matvec_acc_u32": (i32, [u8, u8, u64, u64, vp, vp, vp, vp, vp, vp]),
        "fvb_synth_state": (i32, [u32, u8, u64, u64, u64, pp, vp]),
        "fvb_synth_uniform": (i32, [u8, u64, u64, u64, ctypes.c_double, ctypes.c_double, vp,
                                    vp]),
        "fvb_lookup": (i32, [ctypes.c_char_p, ctypes.POINTER(KernelStruct)]),
        "fvb_emit_source": (i32, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t,
                                  ctypes.POINTER(ctypes.c_size_t)]),
        "fvb_nvrtc_compile": (i32, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_size_t)]),
        "fvb_pattern_count": (u32, []),
        "fvb_pattern": (ctypes.c_char_p, [u32, ctypes.POINTER(ctypes.c_char_p)]),
        "fvb_ctx_create": (i32, [i32, u64, ctypes.POINTER(vp)]),
        "fvb_ctx_destroy": (i32, [vp]),
        "fvb_flux_host": (i32, [vp, gas, u32, u8, u64, pp, pp]),
        "fvb_jacobian_host": (i32, [vp, gas, u32, u8, u64, pp, pp,
                                    ctypes.POINTER(ctypes.c_double)]),
        "fvb_launch_host": (i32, [vp, ctypes.POINTER(KernelStruct), u64, pp, vp, vp,
                                  ctypes.POINTER(ctypes.c_double), vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def lib():
    """The loaded libfvb.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = lib_path()
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (make -C paper_1809_09851_b200/csrc); there is no CPU fallback")
            L = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
            _declare(L)
            _lib = L
    return _lib


def check(status: int) -> None:
    if status == FVB_OK:
        return
    msg = lib().fvb_last_error().decode(errors="replace")
    raise _ERRORS.get(status, FvbError)(status, msg)


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(len(ptrs), 1))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr

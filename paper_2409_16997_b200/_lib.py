"""Loader for the native library ``lib/libifa_b200.so`` (include/ifa_b200.h).

There is deliberately no fallback: if the sm_100a library is missing or
cannot be loaded, every product entry point raises ``NativeLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# IFA_B200_LIB: load an alternative build (A/B timing of kernel variants)
LIB_PATH = os.environ.get("IFA_B200_LIB") or os.path.join(_HERE, "lib", "libifa_b200.so")

IFA_OK = 0
IFA_EINVAL = 22
IFA_EOVERFLOW = 75
IFA_ENOTSUP = 95
IFA_ECUDA = 1000
IFA_EFORMAT = 74

FLAG_SQRT_D = 1
FLAG_CAUSAL = 2
FLAG_FAST = 4
FLAG_DUMP_S = 8

# Every symbol include/ifa_b200.h declares.
EXPORTED_SYMBOLS = (
    "ifa_quantize_per_row",
    "ifa_quantize_per_tensor",
    "ifa_int_flash_fwd",
    "ifa_int_flash_fwd_dump",
    "ifa_int8_attention_step",
    "ifa_half_int8_fwd",
    "ifa_convert_f16",
    "ifa_quantize_per_tensor_v16",
    "ifa_int_flash_fwd_v16",
    "ifa_fp8_quantize_per_tensor",
    "ifa_fp8_attention_fwd",
    "ifa_quantize_per_row_host",
    "ifa_quantize_per_tensor_host",
    "ifa_int_flash_fwd_host",
    "ifa_full_int8_attention_host",
    "ifa_half_int8_fwd_host",
    "ifa_fp8_emulated_attention_host",
    "ifa_tensor_save",
    "ifa_tensor_info",
    "ifa_tensor_load",
    "ifa_audit_init",
    "ifa_code_bounds",
    "ifa_last_error",
    "ifa_version",
)


class NativeLibraryError(RuntimeError):
    pass


class FormatError(RuntimeError):
    """Malformed IFA1 tensor file (ifa::FormatError, tensor_io.hpp:16-20)."""


class PCodeAuditC(C.Structure):
    """Mirror of ``ifa_pcode_audit`` (include/ifa_b200.h)."""

    _fields_ = [("min_code", C.c_int32), ("max_code", C.c_int32),
                ("row_max_block_hits_127", C.c_int32), ("reserved", C.c_int32),
                ("rows_audited", C.c_int64)]


_lib = None


def load() -> C.CDLL:
    """Load (once) and return the native library, or raise loudly."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback")
    try:
        lib = C.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    vp, i64, u32 = C.c_void_p, C.c_int64, C.c_uint32
    lib.ifa_quantize_per_row.argtypes = [vp, i64, i64, vp, vp, vp, vp]
    lib.ifa_quantize_per_row.restype = C.c_int
    lib.ifa_quantize_per_tensor.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp, vp]
    lib.ifa_quantize_per_tensor.restype = C.c_int
    lib.ifa_int_flash_fwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64,
                                      u32, vp, vp]
    lib.ifa_int_flash_fwd.restype = C.c_int
    lib.ifa_int_flash_fwd_dump.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64,
                                           i64, u32, vp, vp, vp]
    lib.ifa_int_flash_fwd_dump.restype = C.c_int
    lib.ifa_int8_attention_step.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                            u32, i64, i64, i64, i64, i64, u32, vp]
    lib.ifa_int8_attention_step.restype = C.c_int
    lib.ifa_half_int8_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, u32, vp]
    lib.ifa_half_int8_fwd.restype = C.c_int
    lib.ifa_convert_f16.argtypes = [vp, i64, vp, vp]
    lib.ifa_convert_f16.restype = C.c_int
    lib.ifa_quantize_per_tensor_v16.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp]
    lib.ifa_quantize_per_tensor_v16.restype = C.c_int
    lib.ifa_int_flash_fwd_v16.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64,
                                          i64, u32, vp]
    lib.ifa_int_flash_fwd_v16.restype = C.c_int
    lib.ifa_fp8_quantize_per_tensor.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp]
    lib.ifa_fp8_quantize_per_tensor.restype = C.c_int
    lib.ifa_fp8_attention_fwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64,
                                          u32, vp]
    lib.ifa_fp8_attention_fwd.restype = C.c_int
    lib.ifa_quantize_per_row_host.argtypes = [vp, i64, i64, vp, vp, vp, vp]
    lib.ifa_quantize_per_row_host.restype = C.c_int
    lib.ifa_quantize_per_tensor_host.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp]
    lib.ifa_quantize_per_tensor_host.restype = C.c_int
    lib.ifa_int_flash_fwd_host.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64,
                                           u32, vp, vp]
    lib.ifa_int_flash_fwd_host.restype = C.c_int
    lib.ifa_full_int8_attention_host.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, i64, u32,
                                                 vp]
    lib.ifa_full_int8_attention_host.restype = C.c_int
    lib.ifa_half_int8_fwd_host.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, u32,
                                           vp]
    lib.ifa_half_int8_fwd_host.restype = C.c_int
    lib.ifa_fp8_emulated_attention_host.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, i64,
                                                    u32, vp]
    lib.ifa_fp8_emulated_attention_host.restype = C.c_int
    i32 = C.c_int32
    lib.ifa_tensor_save.argtypes = [C.c_char_p, i32, vp, i64, i64]
    lib.ifa_tensor_save.restype = C.c_int
    lib.ifa_tensor_info.argtypes = [C.c_char_p, C.POINTER(i32), C.POINTER(i64), C.POINTER(i64)]
    lib.ifa_tensor_info.restype = C.c_int
    lib.ifa_tensor_load.argtypes = [C.c_char_p, i32, vp, i64, i64]
    lib.ifa_tensor_load.restype = C.c_int
    lib.ifa_audit_init.argtypes = [vp, vp]
    lib.ifa_audit_init.restype = C.c_int
    lib.ifa_code_bounds.argtypes = [vp]
    lib.ifa_code_bounds.restype = C.c_int
    lib.ifa_last_error.argtypes = []
    lib.ifa_last_error.restype = C.c_char_p
    lib.ifa_version.argtypes = []
    lib.ifa_version.restype = C.c_char_p
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if rc == IFA_OK:
        return
    msg = load().ifa_last_error().decode(errors="replace")
    if rc == IFA_EINVAL:
        raise ValueError(msg)          # std::invalid_argument
    if rc == IFA_EOVERFLOW:
        raise OverflowError(msg)       # std::overflow_error
    if rc == IFA_EFORMAT:
        raise FormatError(msg)         # ifa::FormatError
    if rc == IFA_ENOTSUP:
        raise NotImplementedError(msg)
    raise NativeLibraryError(f"CUDA failure ({rc}): {msg}")

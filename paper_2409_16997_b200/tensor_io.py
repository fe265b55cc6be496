"""IFA1 tensor files through the C-ABI.

Mirrors ``ifa::save_tensor`` / ``load_tensor`` / ``load_float_tensor`` /
``load_int8_tensor`` (include/ifa/tensor_io.hpp:27-39): host numpy arrays in
and out, ``FormatError`` with the reference's messages for malformed files.
The command-line front end over the same entry points is
``paper_2409_16997_b200/lib/ifa_b200`` (``quantize`` / ``info``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import FormatError  # noqa: F401

_DTYPES = {np.dtype(np.float32): 0, np.dtype(np.int8): 1, np.dtype(np.int32): 2}
_NP = {0: np.float32, 1: np.int8, 2: np.int32}


def save_tensor(matrix: np.ndarray, path: str) -> None:
    m = np.ascontiguousarray(matrix)
    if m.ndim != 2 or m.dtype not in _DTYPES:
        raise ValueError("save_tensor: expected a 2-D float32 / int8 / int32 array")
    lib = _lib.load()
    _lib.check(lib.ifa_tensor_save(path.encode(), _DTYPES[m.dtype], m.ctypes.data,
                                   m.shape[0], m.shape[1]))


def tensor_info(path: str):
    """(dtype, rows, cols) after validating the whole file."""
    lib = _lib.load()
    dt, r, c = C.c_int32(), C.c_int64(), C.c_int64()
    _lib.check(lib.ifa_tensor_info(path.encode(), C.byref(dt), C.byref(r), C.byref(c)))
    return np.dtype(_NP[dt.value]), r.value, c.value


def load_tensor(path: str, expect=None) -> np.ndarray:
    """Any dtype (``expect=None``) or exactly ``expect`` (load_float_tensor /
    load_int8_tensor semantics)."""
    dtype, rows, cols = tensor_info(path)
    want = -1 if expect is None else _DTYPES[np.dtype(expect)]
    out = np.empty((rows, cols), dtype=dtype if expect is None else expect)
    lib = _lib.load()
    _lib.check(lib.ifa_tensor_load(path.encode(), want, out.ctypes.data if out.size else None,
                                   rows, cols))
    return out


def load_float_tensor(path: str) -> np.ndarray:
    return load_tensor(path, np.float32)


def load_int8_tensor(path: str) -> np.ndarray:
    return load_tensor(path, np.int8)

"""IFA1 tensor files: this build's C-ABI reader/writer
against the reference's own tensor_io (oracle/_ref), and the malformed-file
cases of proj/tests/test_tensors.cpp:107-152 with the same messages.
CPU only (file I/O); the GPU `quantize` CLI is in test_gpu_cli.py."""
import ctypes as C
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2409_16997_b200", "lib", "ifa_b200")


def _ref_load(reference, path):
    lib = reference.lib
    lib.ifa_ref_load_tensor.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.c_void_p, C.c_int64]
    dt, r, c = C.c_int(), C.c_int64(), C.c_int64()
    buf = np.empty(1 << 20, np.uint8)
    rc = lib.ifa_ref_load_tensor(path.encode(), C.byref(dt), C.byref(r), C.byref(c),
                                 buf.ctypes.data, buf.size)
    if rc:
        return None, lib.ifa_ref_last_error().decode()
    dtype = {0: np.float32, 1: np.int8, 2: np.int32}[dt.value]
    n = r.value * c.value * np.dtype(dtype).itemsize
    return buf[:n].view(dtype).reshape(r.value, c.value), None


@pytest.mark.parametrize("dtype,shape", [(np.float32, (5, 7)), (np.int8, (3, 128)),
                                         (np.int32, (1, 1)), (np.float32, (0, 4))])
def test_round_trip_and_reference_compat(tmp_path, reference, dtype, shape):
    from paper_2409_16997_b200 import tensor_io
    rng = np.random.default_rng(1)
    m = (rng.standard_normal(shape) * 100).astype(dtype)
    ours = str(tmp_path / "ours.ifa")
    tensor_io.save_tensor(m, ours)
    assert np.array_equal(tensor_io.load_tensor(ours), m)
    got, err = _ref_load(reference, ours)            # reference reads ours
    assert err is None and np.array_equal(got, m)
    theirs = str(tmp_path / "theirs.ifa")
    reference.lib.ifa_ref_save_tensor.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_int64,
                                                  C.c_int64]
    code = {np.float32: 0, np.int8: 1, np.int32: 2}[dtype]
    mm = np.ascontiguousarray(m)
    assert reference.lib.ifa_ref_save_tensor(theirs.encode(), code, mm.ctypes.data,
                                             shape[0], shape[1]) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()   # byte-identical files


def _write(path, data):
    with open(path, "wb") as f:
        f.write(data)


def _header(dtype=0, rows=2, cols=2, magic=b"IFA1", reserved=b"\0\0\0"):
    return magic + bytes([dtype]) + reserved + struct.pack("<QQ", rows, cols)


MALFORMED = [
    ("truncated header", b"IFA1\0\0"),
    ("bad magic", _header(magic=b"IFA2") + b"\0" * 16),
    ("reserved", _header(reserved=b"\0\1\0") + b"\0" * 16),
    ("truncated payload", _header() + b"\0" * 15),
    ("oversized", _header() + b"\0" * 17),
    ("dtype", _header(dtype=7) + b"\0" * 16),
    ("overflow", _header(rows=1 << 40, cols=1 << 40)),
]


@pytest.mark.parametrize("what,data", MALFORMED)
def test_malformed_files_rejected_like_the_reference(tmp_path, reference, what, data):
    from paper_2409_16997_b200 import tensor_io
    path = str(tmp_path / "bad.ifa")
    _write(path, data)
    with pytest.raises(tensor_io.FormatError) as ours:
        tensor_io.load_tensor(path)
    _, theirs = _ref_load(reference, path)
    assert what in str(ours.value)
    assert str(ours.value) == theirs


def test_typed_loaders_and_missing_file(tmp_path):
    from paper_2409_16997_b200 import tensor_io
    path = str(tmp_path / "f.ifa")
    tensor_io.save_tensor(np.ones((2, 2), np.float32), path)
    with pytest.raises(tensor_io.FormatError, match="expected i8 tensor"):
        tensor_io.load_int8_tensor(path)
    with pytest.raises(tensor_io.FormatError, match="cannot open"):
        tensor_io.load_tensor(str(tmp_path / "nope.ifa"))


def test_cli_info_and_usage(tmp_path):
    from paper_2409_16997_b200 import tensor_io
    path = str(tmp_path / "x.ifa")
    tensor_io.save_tensor(np.array([[1, -3], [7, 2]], np.int8), path)
    r = subprocess.run([CLI, "info", path], capture_output=True, text=True)
    assert r.returncode == 0
    assert r.stdout == f"{path}: i8 2x2\nmin -3 max 7\n"
    assert subprocess.run([CLI], capture_output=True).returncode == 2
    assert subprocess.run([CLI, "quantize", "only-one"], capture_output=True).returncode == 2
    bad = str(tmp_path / "bad.ifa")
    _write(bad, b"junk")
    r = subprocess.run([CLI, "info", bad], capture_output=True, text=True)
    assert r.returncode == 1 and "truncated header" in r.stderr

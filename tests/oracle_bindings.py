"""ctypes bindings to the CPU checkers (TEST INFRASTRUCTURE ONLY).

- ``Oracle``: oracle/libifa_oracle.so, the C restatement of the reference
  hot path (oracle/ifa_oracle.c, every function cites reference file:line).
- ``Reference``: oracle/_ref/libifa_ref.so, the UNMODIFIED reference sources
  (/root/reference/proj/src) compiled by oracle/Makefile plus the extern "C"
  shim oracle/ref_shim.cpp.  Absent on a box where it was not prebuilt.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "libifa_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libifa_ref.so")

FLAG_SQRT_D = 1
FLAG_CAUSAL = 2

_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class Audit(C.Structure):
    _fields_ = [("min_code", C.c_int32), ("max_code", C.c_int32),
                ("row_max_block_hits_127", C.c_int32), ("pad_", C.c_int32),
                ("rows_audited", C.c_int64)]

    def as_tuple(self):
        return (self.min_code, self.max_code, bool(self.row_max_block_hits_127),
                self.rows_audited)


def _i8(a):
    return np.ascontiguousarray(a, dtype=np.int8)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Oracle:
    """The C restatement (always buildable: `make -C oracle`)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", os.path.dirname(path), "all"])
        L = self.lib = C.CDLL(path)
        L.ifa_or_expf.restype = C.c_float
        L.ifa_or_expf.argtypes = [C.c_float]
        L.ifa_or_stream_seed.restype = C.c_uint64
        L.ifa_or_stream_seed.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int64, C.c_int64]
        L.ifa_or_generate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_uint64,
                                      C.c_int64, C.c_int64, _f32p]
        L.ifa_or_quantize_per_row.argtypes = [_f32p, C.c_int64, C.c_int64, _i8p, _f32p,
                                              C.POINTER(C.c_int64)]
        L.ifa_or_quantize_per_tensor.argtypes = [_f32p, C.c_int64, C.c_int64, _i8p,
                                                 C.POINTER(C.c_float), C.POINTER(C.c_int64)]
        L.ifa_or_int_gemm_nt.argtypes = [_i8p, _i8p, C.c_int64, C.c_int64, C.c_int64, _i32p]
        L.ifa_or_int_flash_attention.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, C.c_float, C.c_int64, C.c_int64, C.c_int64,
            C.c_int64, C.c_uint32, _f32p, C.POINTER(Audit)]
        L.ifa_or_int_flash_attention_pcodes.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, C.c_float, C.c_int64, C.c_int64, C.c_int64,
            C.c_int64, C.c_uint32, _f32p, C.c_void_p]
        L.ifa_or_int_flash_attention_rows.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, C.c_float, C.c_int64, C.c_int64, C.c_int64,
            C.c_int64, C.c_uint32, C.c_int64, C.c_int64, _f32p]
        L.ifa_or_int_flash_attention_batched.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, _f32p, C.c_int64, C.c_int64, C.c_int64,
            C.c_int64, C.c_int64, C.c_uint32, _f32p, C.c_int]
        L.ifa_or_untiled_int8_attention.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, C.c_float, C.c_int64, C.c_int64, C.c_uint32, _f32p]
        L.ifa_or_reference_attention.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64,
                                                 C.c_int64, C.c_int64, C.c_uint32, _f32p]
        L.ifa_or_half_int8_attention.argtypes = [_i8p, _f32p, _i8p, _f32p, _f32p, C.c_int64,
                                                 C.c_int64, C.c_int64, C.c_int64, C.c_uint32,
                                                 _f32p]
        L.ifa_or_e4m3_encode.restype = C.c_uint8
        L.ifa_or_e4m3_encode.argtypes = [C.c_float]
        L.ifa_or_e4m3_decode.restype = C.c_float
        L.ifa_or_e4m3_decode.argtypes = [C.c_uint8]
        L.ifa_or_fp8_roundtrip.argtypes = [_f32p, C.c_int64, _f32p, C.c_void_p,
                                           C.POINTER(C.c_float)]
        L.ifa_or_fp8_attention.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_uint32, _f32p]
        L.ifa_or_error_accum.argtypes = [_f32p, _f32p, C.c_int64, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
        L.ifa_or_fnv1a64.restype = C.c_uint64
        L.ifa_or_fnv1a64.argtypes = [C.c_void_p, C.c_int64]

    # -- inputs ---------------------------------------------------------
    def stream_seed(self, base, seed_idx, role, b, h):
        return self.lib.ifa_or_stream_seed(base, seed_idx, role, b, h)

    def generate(self, dist, rows, cols, seed, a=None, b=None):
        """dist: 'normal' (N(0,1)) or 'uniform' (U(-0.5,0.5)), eval.cpp:46-51."""
        if dist == "normal":
            d, a, b = 0, 0.0 if a is None else a, 1.0 if b is None else b
        else:
            d, a, b = 1, -0.5 if a is None else a, 0.5 if b is None else b
        out = np.empty((rows, cols), np.float32)
        rc = self.lib.ifa_or_generate(d, a, b, seed, rows, cols, out)
        if rc:
            raise ValueError("generate: bad spec")
        return out

    def slice_inputs(self, dist, n, d, seed=0, seed_idx=0, b=0, h=0):
        """Q, K, V for one (b,h) slice exactly as run_group/run_speed_benchmark
        draw them (eval.cpp:169-180, :341-353)."""
        return tuple(self.generate(dist, n, d, self.stream_seed(seed, seed_idx, role, b, h))
                     for role in range(3))

    # -- quantize -------------------------------------------------------
    def quantize_per_row(self, x):
        x = _f32(x)
        rows, cols = x.shape
        codes = np.empty((rows, cols), np.int8)
        scales = np.empty(rows, np.float32)
        bad = C.c_int64(-1)
        if self.lib.ifa_or_quantize_per_row(x, rows, cols, codes, scales, C.byref(bad)):
            raise ValueError(f"quantize_per_row: non-finite input at index {bad.value}")
        return codes, scales

    def quantize_per_tensor(self, x):
        x = _f32(x)
        rows, cols = x.shape
        codes = np.empty((rows, cols), np.int8)
        scale = C.c_float(0)
        bad = C.c_int64(-1)
        if self.lib.ifa_or_quantize_per_tensor(x, rows, cols, codes, C.byref(scale),
                                               C.byref(bad)):
            raise ValueError(f"quantize_per_tensor: non-finite input at index {bad.value}")
        return codes, np.float32(scale.value)

    def int_gemm_nt(self, a, b):
        a, b = _i8(a), _i8(b)
        out = np.empty((a.shape[0], b.shape[0]), np.int32)
        self.lib.ifa_or_int_gemm_nt(a, b, a.shape[0], b.shape[0], a.shape[1], out)
        return out

    # -- attention ------------------------------------------------------
    def int_flash_attention(self, q, sq, k, sk, v, sv, br=64, bc=64, flags=0, audit=False):
        q, k, v = _i8(q), _i8(k), _i8(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        au = Audit()
        rc = self.lib.ifa_or_int_flash_attention(q, _f32(sq), k, _f32(sk), v, float(sv), n, d,
                                                 br, bc, flags, out, C.byref(au))
        if rc == -2:
            raise OverflowError("int gemm depth exceeds 133144")
        if rc:
            raise ValueError("int_flash_attention: invalid argument")
        return (out, au.as_tuple()) if audit else out

    def int_flash_pcodes(self, q, sq, k, sk, v, sv, br=128, bc=128, flags=0):
        """(O, P codes [n][n] uint8) of int_flash_attention (attention.cpp:299-312)."""
        q, k, v = _i8(q), _i8(k), _i8(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        codes = np.zeros((n, n), np.uint8)
        rc = self.lib.ifa_or_int_flash_attention_pcodes(
            q, _f32(sq), k, _f32(sk), v, float(sv), n, d, br, bc, flags, out,
            codes.ctypes.data_as(C.c_void_p))
        if rc:
            raise ValueError("int_flash_pcodes: invalid argument")
        return out, codes

    def int_flash_rows(self, q, sq, k, sk, v, sv, row_begin, row_end, br=128, bc=128,
                       flags=0):
        """Rows [row_begin, row_end) of int_flash_attention's O (row blocks are
        independent, attention.cpp:267); the other rows of the result are NaN."""
        q, k, v = _i8(q), _i8(k), _i8(v)
        n, d = q.shape
        out = np.full((n, d), np.nan, np.float32)
        if self.lib.ifa_or_int_flash_attention_rows(q, _f32(sq), k, _f32(sk), v, float(sv), n,
                                                    d, br, bc, flags, row_begin, row_end, out):
            raise ValueError("int_flash_rows: invalid argument")
        return out

    def int_flash_attention_batched(self, q, sq, k, sk, v, sv, br=128, bc=128, flags=0,
                                    threads=None):
        q, k, v = _i8(q), _i8(k), _i8(v)
        s, n, d = q.shape
        out = np.empty((s, n, d), np.float32)
        rc = self.lib.ifa_or_int_flash_attention_batched(
            q, _f32(sq), k, _f32(sk), v, _f32(sv), s, n, d, br, bc, flags, out,
            threads or os.cpu_count())
        if rc:
            raise ValueError("int_flash_attention_batched failed")
        return out

    def untiled(self, q, sq, k, sk, v, sv, flags=0):
        q, k, v = _i8(q), _i8(k), _i8(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        if self.lib.ifa_or_untiled_int8_attention(q, _f32(sq), k, _f32(sk), v, float(sv), n,
                                                  d, flags, out):
            raise ValueError("untiled: invalid argument")
        return out

    def half_int8_attention(self, q, sq, k, sk, v, br=64, bc=64, flags=0):
        q, k = _i8(q), _i8(k)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        rc = self.lib.ifa_or_half_int8_attention(q, _f32(sq), k, _f32(sk), _f32(v), n, d, br,
                                                 bc, flags, out)
        if rc:
            raise ValueError("half_int8_attention: invalid argument")
        return out

    def e4m3_encode(self, x):
        return self.lib.ifa_or_e4m3_encode(float(x))

    def e4m3_decode(self, b):
        return self.lib.ifa_or_e4m3_decode(int(b))

    def fp8_roundtrip(self, x):
        """fp8.cpp:78-97 over the whole array: (restored, e4m3 codes, scale s)."""
        x = _f32(x)
        out = np.empty(x.shape, np.float32)
        codes = np.empty(x.shape, np.uint8)
        sc = C.c_float(0.0)
        if self.lib.ifa_or_fp8_roundtrip(x, x.size, out, codes.ctypes.data, C.byref(sc)):
            raise ValueError("fp8_e4m3_roundtrip: non-finite input")
        return out, codes, sc.value

    def fp8_attention(self, q, k, v, br=64, bc=64, flags=0):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        if self.lib.ifa_or_fp8_attention(q, k, v, n, d, br, bc, flags, out):
            raise ValueError("fp8_emulated_attention: invalid argument")
        return out

    def reference_attention(self, q, k, v, flags=0):
        q, k, v = _f32(q), _f32(k), _f32(v)
        out = np.empty((q.shape[0], v.shape[1]), np.float32)
        self.lib.ifa_or_reference_attention(q, k, v, q.shape[0], k.shape[0], q.shape[1],
                                            v.shape[1], flags, out)
        return out

    def error_accum(self, reference, candidate, num=0.0, den=0.0):
        r, c = _f32(reference).ravel(), _f32(candidate).ravel()
        nu, de = C.c_double(num), C.c_double(den)
        self.lib.ifa_or_error_accum(r, c, r.size, C.byref(nu), C.byref(de))
        return nu.value, de.value

    def mre(self, reference, candidate):
        nu, de = self.error_accum(reference, candidate)
        return nu / de

    def fnv1a64(self, arr) -> str:
        a = np.ascontiguousarray(arr)
        return "%016x" % self.lib.ifa_or_fnv1a64(a.ctypes.data, a.nbytes)


class Reference:
    """The unmodified reference library (oracle/_ref/libifa_ref.so)."""

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ifa_ref_last_error.restype = C.c_char_p
        L.ifa_ref_generate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_uint64,
                                       C.c_int64, C.c_int64, _f32p]
        L.ifa_ref_quantize_per_row.argtypes = [_f32p, C.c_int64, C.c_int64, _i8p, _f32p]
        L.ifa_ref_quantize_per_tensor.argtypes = [_f32p, C.c_int64, C.c_int64, _i8p,
                                                  C.POINTER(C.c_float)]
        L.ifa_ref_int_gemm_nt.argtypes = [_i8p, _i8p, C.c_int64, C.c_int64, C.c_int64, _i32p]
        L.ifa_ref_int_flash_attention.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, C.c_float, C.c_int64, C.c_int64, C.c_int64,
            C.c_int64, C.c_int, _f32p, _i64p]
        L.ifa_ref_int_flash_attention_batched.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, _f32p, C.c_int64, C.c_int64, C.c_int64,
            C.c_int64, C.c_int64, _f32p, C.c_int]
        L.ifa_ref_untiled_int8_attention.argtypes = [
            _i8p, _f32p, _i8p, _f32p, _i8p, C.c_float, C.c_int64, C.c_int64, C.c_int, _f32p]
        L.ifa_ref_reference_attention.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64,
                                                  _f32p]
        L.ifa_ref_half_int8_attention.argtypes = [_i8p, _f32p, _i8p, _f32p, _f32p, C.c_int64,
                                                  C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                                  _f32p]
        L.ifa_ref_fp8_roundtrip.argtypes = [_f32p, C.c_int64, C.c_int64, _f32p]
        L.ifa_ref_e4m3_encode.restype = C.c_uint8
        L.ifa_ref_e4m3_encode.argtypes = [C.c_float]
        L.ifa_ref_fp8_attention.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64,
                                            C.c_int64, C.c_int64, C.c_int, _f32p]
        L.ifa_ref_expf.restype = C.c_float
        L.ifa_ref_expf.argtypes = [C.c_float]

    def _check(self, rc):
        if rc == -2:
            raise OverflowError(self.lib.ifa_ref_last_error().decode())
        if rc:
            raise ValueError(self.lib.ifa_ref_last_error().decode())

    def generate(self, dist, rows, cols, seed):
        d, a, b = (0, 0.0, 1.0) if dist == "normal" else (1, -0.5, 0.5)
        out = np.empty((rows, cols), np.float32)
        self._check(self.lib.ifa_ref_generate(d, a, b, seed, rows, cols, out))
        return out

    def quantize_per_row(self, x):
        x = _f32(x)
        codes = np.empty(x.shape, np.int8)
        scales = np.empty(x.shape[0], np.float32)
        self._check(self.lib.ifa_ref_quantize_per_row(x, x.shape[0], x.shape[1], codes,
                                                      scales))
        return codes, scales

    def quantize_per_tensor(self, x):
        x = _f32(x)
        codes = np.empty(x.shape, np.int8)
        scale = C.c_float(0)
        self._check(self.lib.ifa_ref_quantize_per_tensor(x, x.shape[0], x.shape[1], codes,
                                                         C.byref(scale)))
        return codes, np.float32(scale.value)

    def int_gemm_nt(self, a, b):
        a, b = _i8(a), _i8(b)
        out = np.empty((a.shape[0], b.shape[0]), np.int32)
        self._check(self.lib.ifa_ref_int_gemm_nt(a, b, a.shape[0], b.shape[0], a.shape[1],
                                                 out))
        return out

    def int_flash_attention(self, q, sq, k, sk, v, sv, br=64, bc=64, sqrt_d=False,
                            audit=False):
        q, k, v = _i8(q), _i8(k), _i8(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        au = np.zeros(4, np.int64)
        self._check(self.lib.ifa_ref_int_flash_attention(q, _f32(sq), k, _f32(sk), v,
                                                         float(sv), n, d, br, bc,
                                                         int(sqrt_d), out, au))
        if audit:
            return out, (int(au[0]), int(au[1]), bool(au[2]), int(au[3]))
        return out

    def int_flash_attention_batched(self, q, sq, k, sk, v, sv, br=128, bc=128,
                                    threads=None):
        q, k, v = _i8(q), _i8(k), _i8(v)
        s, n, d = q.shape
        out = np.empty((s, n, d), np.float32)
        self._check(self.lib.ifa_ref_int_flash_attention_batched(
            q, _f32(sq), k, _f32(sk), v, _f32(sv), s, n, d, br, bc, out,
            threads or os.cpu_count()))
        return out

    def untiled(self, q, sq, k, sk, v, sv, sqrt_d=False):
        q, k, v = _i8(q), _i8(k), _i8(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        self._check(self.lib.ifa_ref_untiled_int8_attention(q, _f32(sq), k, _f32(sk), v,
                                                            float(sv), n, d, int(sqrt_d),
                                                            out))
        return out

    def reference_attention(self, q, k, v):
        q, k, v = _f32(q), _f32(k), _f32(v)
        out = np.empty(q.shape, np.float32)
        self._check(self.lib.ifa_ref_reference_attention(q, k, v, q.shape[0], q.shape[1],
                                                         out))
        return out

    def expf(self, x):
        return self.lib.ifa_ref_expf(float(x))

    def e4m3_encode(self, x):
        return self.lib.ifa_ref_e4m3_encode(float(x))

    def fp8_roundtrip(self, x):
        x = _f32(x)
        out = np.empty(x.shape, np.float32)
        self._check(self.lib.ifa_ref_fp8_roundtrip(x, x.shape[0], x.shape[1], out))
        return out

    def fp8_attention(self, q, k, v, br=64, bc=64, sqrt_d=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        self._check(self.lib.ifa_ref_fp8_attention(q, k, v, n, d, br, bc, int(sqrt_d), out))
        return out

    def half_int8_attention(self, q, sq, k, sk, v, br=64, bc=64, sqrt_d=False):
        q, k = _i8(q), _i8(k)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        self._check(self.lib.ifa_ref_half_int8_attention(q, _f32(sq), k, _f32(sk), _f32(v), n, d,
                                                         br, bc, int(sqrt_d), out))
        return out

"""The host-buffer C-ABI entry points (include/ifa_b200.h *_host) as a
chunked three-stream pipeline: results must not depend on the chunking, on
pageable vs pinned caller memory, or on the kernel chosen, and must equal
the oracle (pinned bitwise to the reference) -- bitwise in exact mode.

IFA_B200_HOST_CHUNK forces small chunks so a small problem runs through many
pipeline slots (slot reuse, drain order, the audit folded over chunks)."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _p(a):
    if isinstance(a, torch.Tensor):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _case(oracle, slices, n, d, dist="normal"):
    xs = [np.stack([oracle.slice_inputs(dist, n, d, seed=10 * s + 1)[r] for s in range(slices)])
          for r in range(3)]
    codes = []
    for s in range(slices):
        qc, qs = oracle.quantize_per_row(xs[0][s])
        kc, ks = oracle.quantize_per_row(xs[1][s])
        vc, vs = oracle.quantize_per_tensor(xs[2][s])
        codes.append((qc, qs, kc, ks, vc, vs))
    return xs, codes


def _pin(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    assert t.is_pinned()
    return t


@pytest.mark.parametrize("chunk", ["1", "2", "0"])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("fast", [False, True])
def test_int_flash_fwd_host_pipeline(ifa, oracle, monkeypatch, chunk, pinned, fast):
    from paper_2409_16997_b200 import _lib
    monkeypatch.setenv("IFA_B200_HOST_CHUNK", chunk)
    slices, n, d = 5, 256, 64
    _, codes = _case(oracle, slices, n, d)
    arr = [np.ascontiguousarray(np.stack([c[i] for c in codes])) for i in range(5)]
    sv = np.array([c[5] for c in codes], np.float32)
    o = np.zeros((slices, n, d), np.float32)
    bufs = [_pin(a) for a in arr + [sv]] if pinned else arr + [sv]
    out = _pin(o) if pinned else o
    lib = _lib.load()
    flags = _lib.FLAG_FAST if fast else 0
    au = _lib.PCodeAuditC()
    rc = lib.ifa_int_flash_fwd_host(_p(bufs[0]), _p(bufs[1]), _p(bufs[2]), _p(bufs[3]),
                                    _p(bufs[4]), _p(bufs[5]), _p(out), slices, n, d, 64, 128,
                                    flags, None if fast else C.byref(au), None)
    _lib.check(rc)
    got = out.numpy() if pinned else out
    mins, maxs, rows = [], [], 0
    for s, (qc, qs, kc, ks, vc, vs) in enumerate(codes):
        want, a = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 128, audit=True)
        if fast:
            mre = float(np.abs(got[s].astype(np.float64) - want).sum() / np.abs(want).sum())
            assert mre <= 1e-5, (s, mre)
        else:
            assert np.array_equal(got[s].view(np.uint32), want.view(np.uint32)), s
        mins.append(a[0])
        maxs.append(a[1])
        rows += a[3]
    if not fast:
        assert (au.min_code, au.max_code, au.rows_audited) == (min(mins), max(maxs), rows)


@pytest.mark.parametrize("chunk", ["1", "3", "0"])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("n,d", [(256, 128), (200, 64)])
def test_full_int8_attention_host(ifa, oracle, monkeypatch, chunk, pinned, n, d):
    """eval.cpp:98-102's quantize + attention step from f32 host buffers: in
    exact mode bitwise the oracle's codes-then-attention result."""
    from paper_2409_16997_b200 import _lib
    monkeypatch.setenv("IFA_B200_HOST_CHUNK", chunk)
    slices = 4
    xs, codes = _case(oracle, slices, n, d, "uniform")
    o = np.zeros((slices, n, d), np.float32)
    ins = [_pin(x) for x in xs] if pinned else [np.ascontiguousarray(x) for x in xs]
    out = _pin(o) if pinned else o
    lib = _lib.load()
    for flags in (0, _lib.FLAG_FAST):
        _lib.check(lib.ifa_full_int8_attention_host(_p(ins[0]), _p(ins[1]), _p(ins[2]), _p(out),
                                                    slices, n, d, 64, 128, flags, None))
        got = out.numpy() if pinned else out
        for s, (qc, qs, kc, ks, vc, vs) in enumerate(codes):
            want = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 128)
            if flags:
                mre = float(np.abs(got[s].astype(np.float64) - want).sum() / np.abs(want).sum())
                assert mre <= 1e-5, (s, mre)
            else:
                assert np.array_equal(got[s].view(np.uint32), want.view(np.uint32)), s


def test_full_int8_attention_host_rejects_nonfinite(ifa, oracle, monkeypatch):
    from paper_2409_16997_b200 import _lib
    monkeypatch.setenv("IFA_B200_HOST_CHUNK", "1")
    slices, n, d = 3, 128, 64
    xs, _ = _case(oracle, slices, n, d)
    k = np.ascontiguousarray(xs[1])
    k[2, 5, 7] = np.nan
    o = np.zeros((slices, n, d), np.float32)
    lib = _lib.load()
    rc = lib.ifa_full_int8_attention_host(_p(np.ascontiguousarray(xs[0])), _p(k),
                                          _p(np.ascontiguousarray(xs[2])), _p(o), slices, n, d,
                                          64, 64, 0, None)
    assert rc == _lib.IFA_EINVAL
    idx = (2 * n + 5) * d + 7
    assert lib.ifa_last_error().decode() == \
        f"full_int8_attention: k: non-finite input at index {idx}"

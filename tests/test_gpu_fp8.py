"""FP8 e4m3 baseline on the GPU against the oracle.

- fp8_quantize_per_tensor: e4m3 codes and the per-slice scale 448/max|x|
  are BITWISE the reference's fp8_e4m3_roundtrip (fp8.cpp:78-97; the oracle
  restatement is pinned to the reference library in tests/test_oracle.py),
  and the decoded fp16 values are exact.
- fp8_emulated_attention (attention.cpp:401-407): S on tcgen05 kind::f8f6f4
  (f32 accumulate), float softmax, fp16 weights x decoded V.  Tolerance:
  MRE vs the reference <= 2e-3, max|dO| <= 4e-3 * max|V|, and the error
  against fp64 within 1% (+1e-5) of the reference algorithm's own.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("shape", [(1, 2), (33, 8), (256, 64), (4096, 128)])
@pytest.mark.parametrize("dist", ["normal", "uniform"])
def test_fp8_codes_bitwise(ifa, oracle, shape, dist):
    x = oracle.generate(dist, shape[0], shape[1], seed=shape[0] + shape[1])
    t = ifa.fp8_quantize_per_tensor(_dev(x))
    want, codes, s = oracle.fp8_roundtrip(x)
    assert np.array_equal(t.codes.cpu().numpy(), codes)
    assert float(t.scale.item()) == s
    dec = t.decoded.float().cpu().numpy()
    ref_dec = np.array([oracle.e4m3_decode(c) for c in codes.ravel()[:4096]], np.float32)
    assert np.array_equal(dec.ravel()[:4096], ref_dec)
    assert np.array_equal((dec / np.float32(s)).view(np.uint32), want.view(np.uint32))


def test_fp8_codes_edge_values(ifa, oracle):
    """Ties, saturation and subnormals: a probe matrix with max 448 (s = 1)."""
    rng = np.random.default_rng(3)
    vals = [448.0, -448.0, 0.0, -0.0, 2.0 ** -9, 2.0 ** -10, 3 * 2.0 ** -11, 1.0625, 1.1875,
            240.0, 232.0, 2.0 ** -6 * 1.0625, 447.9]
    for e in range(-9, 8):
        for m in range(16):
            vals.append((8 + m / 2.0) * 2.0 ** (e - 3))
    x = np.asarray(vals + list(rng.standard_normal(1000) * 30), np.float32)
    x = np.concatenate([x, -x])[None, :]
    x = x[:, : x.shape[1] // 2 * 2]
    t = ifa.fp8_quantize_per_tensor(_dev(x))
    _, codes, s = oracle.fp8_roundtrip(x)
    assert s == 1.0
    assert np.array_equal(t.codes.cpu().numpy(), codes)


def test_fp8_batched_slices_and_zero_slice(ifa, oracle):
    x = np.random.default_rng(4).standard_normal((3, 64, 32)).astype(np.float32)
    x[1] = 0.0
    t = ifa.fp8_quantize_per_tensor(_dev(x))
    for s_ in range(3):
        _, codes, s = oracle.fp8_roundtrip(x[s_])
        assert np.array_equal(t.codes[s_].cpu().numpy(), codes)
        assert float(t.scale[s_].item()) == s
    with pytest.raises(ValueError, match="non-finite"):
        y = x.copy()
        y[2, 3, 4] = np.inf
        ifa.fp8_quantize_per_tensor(_dev(y))


def _check(oracle, got, want, v):
    assert np.isfinite(got).all()
    mre = oracle.mre(want, got)
    assert mre <= 2e-3, mre
    assert np.abs(got - want).max() <= 4e-3 * max(np.abs(v).max(), 1e-30)


@pytest.mark.parametrize("dist", ["normal", "uniform"])
@pytest.mark.parametrize("n,d,sqrt_d", [(128, 64, False), (200, 64, True), (1024, 64, False),
                                        (96, 128, False), (333, 128, True), (1024, 128, False),
                                        (256, 128, True), (384, 64, True)])
def test_fp8_attention_matches_oracle(ifa, oracle, dist, n, d, sqrt_d):
    q, k, v = oracle.slice_inputs(dist, n, d, seed=19)
    cfg = ifa.AttentionConfig(ifa.BlockSpec(64, 64), apply_sqrt_d_scaling=sqrt_d)
    got = ifa.fp8_emulated_attention(_dev(q), _dev(k), _dev(v), cfg).cpu().numpy()
    want = oracle.fp8_attention(q, k, v, 64, 64, flags=1 if sqrt_d else 0)
    _check(oracle, got, want, v)


@pytest.mark.parametrize("dist,d", [("normal", 64), ("uniform", 128)])
def test_fp8_accuracy_vs_fp64_matches_reference(ifa, oracle, dist, d):
    q, k, v = oracle.slice_inputs(dist, 1024, d, seed=0)
    got = ifa.fp8_emulated_attention(_dev(q), _dev(k), _dev(v)).cpu().numpy()
    want = oracle.fp8_attention(q, k, v, 64, 64)
    exact = oracle.reference_attention(q, k, v)
    e_ref, e_gpu = oracle.mre(exact, want), oracle.mre(exact, got)
    assert e_gpu <= 1.01 * e_ref + 1e-5, (e_gpu, e_ref)


def test_fp8_attention_batched(ifa, oracle):
    b, h, n, d = 2, 2, 256, 128
    rng = np.random.default_rng(9)
    x = [rng.standard_normal((b, h, n, d)).astype(np.float32) for _ in range(3)]
    got = ifa.fp8_emulated_attention(*(_dev(t) for t in x)).cpu().numpy()
    for bi in range(b):
        for hi in range(h):
            want = oracle.fp8_attention(x[0][bi, hi], x[1][bi, hi], x[2][bi, hi], 64, 64)
            _check(oracle, got[bi, hi], want, x[2][bi, hi])


@pytest.mark.parametrize("zero", ["q", "k", "v", "qkv"])
@pytest.mark.parametrize("n", [256, 200])
def test_fp8_attention_zero_slices(ifa, oracle, zero, n):
    """An all-zero Q, K or V slice has e4m3 scale 0: the reference's
    roundtrip returns zeros there (fp8.cpp:78-97), so the scores are 0 (uniform
    weights, O = mean of the restored V) or O = 0 -- never NaN."""
    d = 64
    q, k, v = oracle.slice_inputs("normal", n, d, seed=9)
    for name, t in (("q", q), ("k", k), ("v", v)):
        if name in zero:
            t[:] = 0.0
    got = ifa.fp8_emulated_attention(_dev(q), _dev(k), _dev(v)).cpu().numpy()
    want = oracle.fp8_attention(q, k, v, 64, 64)
    assert np.isfinite(got).all()
    assert np.isfinite(want).all()
    scale = max(float(np.abs(want).max()), 1e-30)
    assert float(np.abs(got - want).max()) <= 4e-3 * max(scale, float(np.abs(v).max())), zero

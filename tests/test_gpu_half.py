"""Half-INT8 attention on the GPU against the oracle.

The reference's half_int8_attention (attention.cpp:359-399) keeps V and the
attention weights in f32; the sm_100a kernel feeds both to the tensor core
as fp16 with f32 accumulation, so the output is checked within a tolerance:

- MRE(GPU, oracle) <= 2e-3, and max|dO| <= 4e-3 * max|V| (fp16 weights and
  V carry 2^-11 relative rounding each; the 16-warp kernel's row sum is the
  tensor core's P.1 over the same fp16 weights, the two-Q-tile kernel
  (n % 128 == 0) sums the f32 weights);
- the GPU's error against the fp64 reference_attention is within 1% (+1e-5)
  of the reference algorithm's own error -- the fp16 steps must not change
  the accuracy the INT8 Q/K quantization sets.
The oracle's half-INT8 restatement is pinned bitwise to the reference
library in tests/test_oracle.py.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MRE_TOL = 2e-3
MAXABS_TOL = 4e-3
ACC_REL = 1.01


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run(ifa, q, k, v, br=64, bc=64, sqrt_d=False):
    qq = ifa.quantize_per_row(_dev(q))
    kq = ifa.quantize_per_row(_dev(k))
    cfg = ifa.AttentionConfig(ifa.BlockSpec(br, bc), apply_sqrt_d_scaling=sqrt_d)
    return ifa.half_int8_attention(qq, kq, _dev(v), cfg), qq, kq


def _oracle(oracle, qq, kq, v, br, bc, sqrt_d):
    return oracle.half_int8_attention(qq.values.cpu().numpy(), qq.scales.cpu().numpy(),
                                      kq.values.cpu().numpy(), kq.scales.cpu().numpy(), v,
                                      br, bc, 1 if sqrt_d else 0)


def _check(oracle, got, want, v):
    assert np.isfinite(got).all()
    mre = oracle.mre(want, got)
    assert mre <= MRE_TOL, mre
    assert np.abs(got - want).max() <= MAXABS_TOL * max(np.abs(v).max(), 1e-30)


@pytest.mark.parametrize("dist", ["normal", "uniform"])
@pytest.mark.parametrize("n,d", [(128, 64), (200, 64), (1024, 64), (96, 128), (333, 128),
                                 (1024, 128)])
def test_half_int8_matches_oracle(ifa, oracle, dist, n, d):
    q, k, v = oracle.slice_inputs(dist, n, d, seed=11)
    got, qq, kq = _run(ifa, q, k, v)
    want = _oracle(oracle, qq, kq, v, 64, 64, False)
    _check(oracle, got.cpu().numpy(), want, v)


@pytest.mark.parametrize("n", [300, 256])  # 256: the two-Q-tile pipeline
@pytest.mark.parametrize("br,bc,sqrt_d", [(64, 64, True), (128, 128, False), (16, 48, True),
                                          (1, 1000, False)])
def test_half_int8_blocks_and_scaling(ifa, oracle, br, bc, sqrt_d, n):
    q, k, v = oracle.slice_inputs("normal", n, 128, seed=5)
    got, qq, kq = _run(ifa, q, k, v, br, bc, sqrt_d)
    want = _oracle(oracle, qq, kq, v, br, bc, sqrt_d)
    _check(oracle, got.cpu().numpy(), want, v)


@pytest.mark.parametrize("dist,d", [("normal", 64), ("uniform", 128)])
def test_half_int8_accuracy_vs_fp64_matches_reference(ifa, oracle, dist, d):
    q, k, v = oracle.slice_inputs(dist, 1024, d, seed=0)
    got, qq, kq = _run(ifa, q, k, v)
    want = _oracle(oracle, qq, kq, v, 64, 64, False)
    exact = oracle.reference_attention(q, k, v)
    e_ref = oracle.mre(exact, want)
    e_gpu = oracle.mre(exact, got.cpu().numpy())
    assert e_gpu <= ACC_REL * e_ref + 1e-5, (e_gpu, e_ref)


def test_half_int8_batched_slices(ifa, oracle):
    b, h, n, d = 2, 3, 160, 64
    rng = np.random.default_rng(7)
    q = rng.standard_normal((b, h, n, d)).astype(np.float32)
    k = rng.standard_normal((b, h, n, d)).astype(np.float32)
    v = rng.standard_normal((b, h, n, d)).astype(np.float32) * 3
    got, qq, kq = _run(ifa, q, k, v)
    got = got.cpu().numpy()
    qc, qs = qq.values.cpu().numpy(), qq.scales.cpu().numpy()
    kc, ks = kq.values.cpu().numpy(), kq.scales.cpu().numpy()
    for bi in range(b):
        for hi in range(h):
            want = oracle.half_int8_attention(qc[bi, hi], qs[bi, hi], kc[bi, hi], ks[bi, hi],
                                              v[bi, hi], 64, 64, 0)
            _check(oracle, got[bi, hi], want, v[bi, hi])


def test_half_int8_zero_query_rows_average_v(ifa, oracle):
    """sQ == 0 rows weigh every key equally (s = 0 for all keys)."""
    q, k, v = oracle.slice_inputs("normal", 256, 64, seed=2)
    q[::7] = 0.0
    got, qq, kq = _run(ifa, q, k, v)
    want = _oracle(oracle, qq, kq, v, 64, 64, False)
    _check(oracle, got.cpu().numpy(), want, v)
    np.testing.assert_allclose(got.cpu().numpy()[0], v.mean(axis=0), atol=2e-3)


def test_half_int8_argument_errors(ifa):
    x = torch.randn(64, 64, device="cuda")
    qq = ifa.quantize_per_row(x)
    with pytest.raises(ValueError, match="k/v row counts differ"):
        ifa.half_int8_attention(qq, qq, x[:32])
    with pytest.raises(ValueError, match="Br and Bc"):
        ifa.half_int8_attention(qq, qq, x, ifa.AttentionConfig(ifa.BlockSpec(0, 64)))
    q48 = ifa.quantize_per_row(torch.randn(64, 48, device="cuda"))
    with pytest.raises(NotImplementedError):
        ifa.half_int8_attention(q48, q48, torch.randn(64, 48, device="cuda"))
    with pytest.raises(NotImplementedError):
        ifa.half_int8_attention(qq, qq, x, ifa.AttentionConfig(causal=True))


def test_half_int8_rejects_v_outside_fp16(ifa, oracle):
    """V reaches the tensor core as fp16: values beyond 65504 are refused
    (ValueError) rather than turned into inf/NaN output."""
    n, d = 128, 64
    q, k, v = oracle.slice_inputs("normal", n, d, seed=4)
    qc, qs = oracle.quantize_per_row(q)
    kc, ks = oracle.quantize_per_row(k)
    v[3, 5] = 1.0e6
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    with pytest.raises(ValueError, match="fp16 range"):
        ifa.half_int8_attention(ifa.QuantizedRows(dev(qc), dev(qs)),
                                ifa.QuantizedRows(dev(kc), dev(ks)), dev(v))

"""Head dims > 128 (VERDICT r1 missing item 6): the reference accepts any d up
to 133144 (include/ifa/gemm.hpp:22, src/attention.cpp:241-242).  On the GPU
they run on attn.cu's general kernel with S accumulated over 128-column depth
chunks of Q and K and one launch per 128-column chunk of O (launch_wide).
Exact mode is compared BITWISE with the oracle (O and the P-code audit), the
tolerance mode against the same bar as every fast-mode kernel."""
import numpy as np
import pytest

from test_gpu_parity import FAST_MRE, _bits, _dev, _fast_close, _gpu_attention, _quantized_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,bc", [(130, 129, 64), (256, 192, 128), (300, 200, 128),
                                    (384, 256, 128), (200, 384, 77), (64, 1000, 64),
                                    (257, 250, 300)])
@pytest.mark.parametrize("dist", ["normal", "uniform"])
def test_wide_bitwise_vs_oracle(ifa, oracle, n, d, bc, dist):
    _, (qc, qs, kc, ks, vc, vs) = _quantized_case(oracle, dist, n, d, seed=n * 7 + d)
    want, wa = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, bc, audit=True)
    got, ga = _gpu_attention(ifa, qc, qs, kc, ks, vc, vs, 64, bc, audit=True)
    assert np.array_equal(_bits(got), _bits(want)), (n, d, bc, float(np.abs(got - want).max()))
    assert ga == wa


@pytest.mark.parametrize("n,d,bc", [(300, 160, 128), (513, 256, 1000)])
def test_wide_causal_and_sqrt_d_bitwise(ifa, oracle, n, d, bc):
    _, (qc, qs, kc, ks, vc, vs) = _quantized_case(oracle, "normal", n, d, seed=d)
    want, wa = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, bc, flags=2, audit=True)
    got, ga = _gpu_attention(ifa, qc, qs, kc, ks, vc, vs, 64, bc, causal=True, audit=True)
    assert np.array_equal(_bits(got), _bits(want))
    assert ga == wa
    want = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, bc, flags=1)
    got = _gpu_attention(ifa, qc, qs, kc, ks, vc, vs, 64, bc, sqrt_d=True)
    assert np.array_equal(_bits(got), _bits(want))


def test_wide_batched_slices_bitwise(ifa, oracle):
    n, d, slices = 256, 320, 3
    parts = [_quantized_case(oracle, "uniform" if s % 2 else "normal", n, d, seed=s)[1]
             for s in range(slices)]
    qc, qs, kc, ks, vc = (np.stack([p[i] for p in parts]) for i in range(5))
    sv = np.array([p[5] for p in parts], np.float32)
    want = oracle.int_flash_attention_batched(qc, qs, kc, ks, vc, sv, 64, 128)
    got = _gpu_attention(ifa, qc, qs, kc, ks, vc, sv, 64, 128)
    assert np.array_equal(_bits(got), _bits(want))


def test_wide_max_depth_int32_edge(ifa, oracle):
    """d = 133144, every code 127: S = 127^2 * d = 2,147,479,576, the largest
    score int32 holds under the reference's depth limit (gemm.cpp:22-28)."""
    n, d = 3, 133144
    qc = np.full((n, d), 127, np.int8)
    kc = np.full((n, d), 127, np.int8)
    qc[1, ::2] = -127                     # a second row with S = 0
    vc = np.tile(np.arange(d, dtype=np.int64) % 255 - 127, (n, 1)).astype(np.int8)
    qs = np.array([1e-9, 2e-9, 3e-9], np.float32)
    ks = np.array([1e-9, 1e-9, 2e-9], np.float32)
    vs = np.float32(0.01)
    want = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 64)
    got = _gpu_attention(ifa, qc, qs, kc, ks, vc, vs, 64, 64)
    assert np.array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("n,d", [(256, 192), (300, 256), (1024, 512)])
@pytest.mark.parametrize("causal", [False, True])
def test_wide_fast_mode_within_tolerance(ifa, oracle, n, d, causal):
    _, (qc, qs, kc, ks, vc, vs) = _quantized_case(oracle, "normal", n, d, seed=n + d)
    want = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 128, flags=2 if causal else 0)
    inputs = ifa.QuantizedAttentionInputs(
        ifa.QuantizedRows(_dev(qc), _dev(qs)), ifa.QuantizedRows(_dev(kc), _dev(ks)),
        ifa.QuantizedTensor(_dev(vc), _dev(np.asarray(vs, np.float32))))
    got = ifa.int_flash_attention(inputs, ifa.AttentionConfig(
        ifa.BlockSpec(64, 128), causal=causal, fast=True)).cpu().numpy()
    mre, mx, bound = _fast_close(got, want, vc, vs)
    assert mre <= FAST_MRE, (mre, mx)
    assert mx <= bound, (mre, mx, bound)


def test_wide_dump_is_refused(ifa):
    import torch
    z = torch.zeros(1, 4, 130, dtype=torch.int8, device="cuda")
    s = torch.ones(1, 4, device="cuda")
    inputs = ifa.QuantizedAttentionInputs(ifa.QuantizedRows(z, s), ifa.QuantizedRows(z, s),
                                          ifa.QuantizedTensor(z, torch.ones(1, device="cuda")))
    with pytest.raises(RuntimeError):
        ifa.int_flash_attention_dump(inputs, ifa.AttentionConfig(ifa.BlockSpec(64, 128),
                                                                 fast=True))

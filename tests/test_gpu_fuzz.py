"""Randomised shapes through the public API against the oracle: every kernel
variant the dispatcher can pick (exact 16-warp generic/fast-path, tolerance
two-Q-tile / quad / 16-warp, causal, 1/sqrt(d), any Bc), batched slices,
ragged n and padded d.  Exact mode must be bitwise; tolerance mode within the
bar of tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

FAST_MRE = 5e-5  # random shapes down to n = 1 (few keys per row); fixed shapes hold 2e-5


def _case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 2, 31, 64, 127, 128, 129, 200, 255, 256, 300, 384, 511, 640]))
    d = int(rng.choice([1, 8, 16, 33, 64, 80, 100, 128]))
    slices = int(rng.integers(1, 4))
    bc = int(rng.choice([1, 7, 32, 64, 100, 128, 200, 1000]))
    causal = bool(rng.integers(0, 2))
    sqrt_d = bool(rng.integers(0, 2))
    fast = bool(rng.integers(0, 2))
    dist = "normal" if rng.integers(0, 2) else "uniform"
    return n, d, slices, bc, causal, sqrt_d, fast, dist


@pytest.mark.parametrize("seed", range(120))
def test_random_shapes_against_oracle(ifa, oracle, seed):
    n, d, slices, bc, causal, sqrt_d, fast, dist = _case(seed)
    flags = (1 if sqrt_d else 0) | (2 if causal else 0)
    xs = []
    for s in range(slices):
        xs.append(oracle.slice_inputs(dist, n, d, seed=seed, b=0, h=s))
    q = np.stack([x[0] for x in xs])
    k = np.stack([x[1] for x in xs])
    v = np.stack([x[2] for x in xs])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    qq, kq, vq = ifa.quantize_per_row(dev(q)), ifa.quantize_per_row(dev(k)), \
        ifa.quantize_per_tensor(dev(v))
    cfg = ifa.AttentionConfig(ifa.BlockSpec(64, bc), apply_sqrt_d_scaling=sqrt_d, causal=causal,
                              fast=fast)
    got = ifa.int_flash_attention(ifa.QuantizedAttentionInputs(qq, kq, vq), cfg).cpu().numpy()
    for s in range(slices):
        qc, qs = oracle.quantize_per_row(q[s])
        kc, ks = oracle.quantize_per_row(k[s])
        vc, vs = oracle.quantize_per_tensor(v[s])
        assert np.array_equal(qq.values[s].cpu().numpy(), qc)
        assert np.array_equal(vq.values[s].cpu().numpy(), vc)
        want = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, bc, flags=flags)
        if fast:
            g = got[s].astype(np.float64)
            mre = float(np.abs(g - want).sum() / max(np.abs(want).sum(), 1e-300))
            bound = 2.0 / 127.0 * float(np.abs(vc).max()) * float(vs)
            assert mre <= FAST_MRE and float(np.abs(g - want).max()) <= bound + 1e-30, \
                (seed, n, d, bc, causal, sqrt_d, mre)
        else:
            assert np.array_equal(got[s].view(np.uint32), want.view(np.uint32)), \
                (seed, n, d, bc, causal, sqrt_d)


@pytest.mark.parametrize("seed", range(30))
def test_random_quantizer_shapes_bitwise(ifa, oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    slices = int(rng.integers(1, 4))
    rows = int(rng.choice([1, 3, 17, 64, 129, 500]))
    cols = int(rng.choice([1, 2, 5, 16, 33, 64, 100, 128, 256]))
    scale = float(rng.choice([1e-30, 1e-3, 1.0, 1e4]))
    x = (rng.standard_normal((slices, rows, cols)) * scale).astype(np.float32)
    if rng.integers(0, 4) == 0:
        x[0] = 0.0  # an all-zero slice: scale 0, codes 0
    xt = torch.from_numpy(x).cuda()
    r = ifa.quantize_per_row(xt)
    t = ifa.quantize_per_tensor(xt)
    for s in range(slices):
        qc, qs = oracle.quantize_per_row(x[s])
        assert np.array_equal(r.values[s].cpu().numpy(), qc)
        assert np.array_equal(r.scales[s].cpu().numpy().view(np.uint32), qs.view(np.uint32))
        vc, vs = oracle.quantize_per_tensor(x[s])
        assert np.array_equal(t.values[s].cpu().numpy(), vc)
        assert np.float32(t.scale[s].item()) == np.float32(vs)


@pytest.mark.parametrize("seed", range(16))
def test_random_float_weight_variants(ifa, oracle, seed):
    """half-INT8 and FP8 (both kernels: n % 128 == 0 runs the two-Q-tile
    pipeline) against their oracle restatements."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.choice([1, 50, 128, 200, 256, 384]))
    d = int(rng.choice([64, 128]))
    sqrt_d = bool(rng.integers(0, 2))
    bc = int(rng.choice([16, 64, 128, 1000]))
    q, k, v = oracle.slice_inputs("normal" if seed % 2 else "uniform", n, d, seed=seed)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    cfg = ifa.AttentionConfig(ifa.BlockSpec(64, bc), apply_sqrt_d_scaling=sqrt_d)
    qq, kq = ifa.quantize_per_row(dev(q)), ifa.quantize_per_row(dev(k))
    got = ifa.half_int8_attention(qq, kq, dev(v), cfg).cpu().numpy()
    want = oracle.half_int8_attention(qq.values.cpu().numpy(), qq.scales.cpu().numpy(),
                                      kq.values.cpu().numpy(), kq.scales.cpu().numpy(), v,
                                      64, bc, 1 if sqrt_d else 0)
    assert oracle.mre(want, got) <= 2e-3
    got8 = ifa.fp8_emulated_attention(dev(q), dev(k), dev(v), cfg).cpu().numpy()
    want8 = oracle.fp8_attention(q, k, v, 64, bc, flags=1 if sqrt_d else 0)
    assert oracle.mre(want8, got8) <= 2e-3

"""At-size parity for the long-sequence BASELINE configs.

C3 (B1 H32 N16384 d128 causal) and C5 (B64 H32 N8192 d128): one slice at the
config's sequence length through the product API, compared with the oracle
(pinned bitwise to the reference in test_oracle.py; the causal restatement
follows attention.cpp:267-351 with the KV loop bounded at the diagonal) on
sampled Q tiles -- the first, a middle one and the last (for causal the last
tile reads every key, the first only its diagonal).  Row blocks of the
reference are independent (attention.cpp:267), so the oracle computes just
those rows (ifa_or_int_flash_attention_rows).

Exact mode: bitwise.  Tolerance mode (the bench default): MRE <= FAST_MRE and
max|dO| <= the reference's multi-block bound 2/127 * max|V| * sV
(verify.cpp:65-70).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

FAST_MRE = 1e-5


def _dev(a):
    a = np.asarray(a)
    if a.ndim == 0:
        return torch.tensor(a.item(), dtype=torch.float32, device="cuda")
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def slices(oracle):
    out = {}
    for name, n in (("c3", 16384), ("c5", 8192)):
        q, k, v = oracle.slice_inputs("normal", n, 128, seed=3 if name == "c3" else 5)
        qc, qs = oracle.quantize_per_row(q)
        kc, ks = oracle.quantize_per_row(k)
        vc, vs = oracle.quantize_per_tensor(v)
        out[name] = (qc, qs, kc, ks, vc, vs)
    return out


@pytest.mark.parametrize("name,causal", [("c3", True), ("c5", False)])
@pytest.mark.parametrize("fast", [True, False])
def test_sampled_q_tiles_at_size(ifa, oracle, slices, name, causal, fast):
    qc, qs, kc, ks, vc, vs = slices[name]
    n = qc.shape[0]
    inputs = ifa.QuantizedAttentionInputs(
        ifa.QuantizedRows(_dev(qc), _dev(qs)), ifa.QuantizedRows(_dev(kc), _dev(ks)),
        ifa.QuantizedTensor(_dev(vc), _dev(np.asarray(vs, np.float32))))
    cfg = ifa.AttentionConfig(ifa.BlockSpec(128, 128), causal=causal, fast=fast)
    got = ifa.int_flash_attention(inputs, cfg).cpu().numpy()
    assert np.isfinite(got).all()
    bound = 2.0 / 127.0 * float(np.abs(vc).max()) * float(vs)
    for r0 in (0, (n // 2 // 128) * 128, n - 128):
        want = oracle.int_flash_rows(qc, qs, kc, ks, vc, vs, r0, r0 + 128, 128, 128,
                                     flags=2 if causal else 0)[r0:r0 + 128]
        g = got[r0:r0 + 128]
        if fast:
            err = np.abs(g.astype(np.float64) - want)
            mre = float(err.sum() / np.abs(want).sum())
            assert mre <= FAST_MRE and float(err.max()) <= bound, (r0, mre, float(err.max()))
        else:
            assert np.array_equal(g.view(np.uint32), want.view(np.uint32)), r0

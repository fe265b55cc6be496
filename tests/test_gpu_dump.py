"""int32 S tiles and P codes of the tolerance-mode kernel vs the reference.

north_star: "int32 S tiles bit-exact".  ``ifa_int_flash_fwd_dump`` runs a
separate instantiation of the full-INT8 tolerance kernel -- the bench-default
two-Q-tile kernel (csrc/attn_pp.cu), or with IFA_B200_WS=1 the
one-row-per-thread kernel (csrc/attn_ws.cu); both are tested -- that writes
every S tile it reads back from the tcgen05 kind::i8 TMEM accumulator, and
every P code it feeds to P.V.

* S is compared BITWISE with the oracle's int_gemm_nt (gemm.cpp:32-46,
  reached from attention.cpp:275-276), with the unmodified reference
  library's int_gemm_nt, and with the committed C1 golden hash
  (tests/golden/c1_known_answers.json).
* P codes are compared with the oracle's codes at the same Bc = 128
  (attention.cpp:299-312).  Tolerance mode computes 127 * exp(.) with one
  MUFU ex2.approx per code, so a code may flip by one where the exact value
  lies within the estimate's error of a .5 boundary: the test reports the
  flip rate and bounds it (|dP| <= 1 everywhere, flips <= 1e-4 of codes).
"""
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["pp", "ws"], autouse=True)
def kernel(request, monkeypatch):
    monkeypatch.setenv("IFA_B200_WS", "1" if request.param == "ws" else "0")
    return request.param

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c1_known_answers.json")
MAX_FLIP_RATE = 1e-4


def _dev(a):
    a = np.asarray(a)
    if a.ndim == 0:
        return torch.tensor(a.item(), dtype=torch.float32, device="cuda")
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _inputs(ifa, qc, qs, kc, ks, vc, vs):
    return ifa.QuantizedAttentionInputs(
        ifa.QuantizedRows(_dev(qc), _dev(qs)), ifa.QuantizedRows(_dev(kc), _dev(ks)),
        ifa.QuantizedTensor(_dev(vc), _dev(np.asarray(vs, np.float32))))


def _case(oracle, dist, n, d, seed=0):
    q, k, v = oracle.slice_inputs(dist, n, d, seed=seed)
    qc, qs = oracle.quantize_per_row(q)
    kc, ks = oracle.quantize_per_row(k)
    vc, vs = oracle.quantize_per_tensor(v)
    return qc, qs, kc, ks, vc, vs


def _computed_tiles_mask(n, causal):
    """[n][n] bool: entries inside the KV tiles the kernel computes."""
    if not causal:
        return np.ones((n, n), bool)
    rows = np.arange(n)[:, None] // 128
    cols = np.arange(n)[None, :] // 128
    return cols <= rows


def _flips(got_p, want_p, mask):
    diff = got_p.astype(np.int32) - want_p.astype(np.int32)
    diff = np.where(mask, diff, 0)
    return int(np.count_nonzero(diff)), int(np.abs(diff).max(initial=0)), int(mask.sum())


@pytest.mark.parametrize("dist", ["normal", "uniform"])
def test_c1_s_tiles_match_golden_and_reference(ifa, oracle, reference, dist):
    """C1 (N=1024, d=64): the full int32 S equals the reference's int_gemm_nt
    bit for bit, and its FNV-1a hash is the committed golden."""
    qc, qs, kc, ks, vc, vs = _case(oracle, dist, 1024, 64)
    _, s, p = ifa.int_flash_attention_dump(_inputs(ifa, qc, qs, kc, ks, vc, vs),
                                           ifa.AttentionConfig(ifa.BlockSpec(128, 128)))
    s = s.cpu().numpy()
    assert np.array_equal(s, oracle.int_gemm_nt(qc, kc))
    assert np.array_equal(s, reference.int_gemm_nt(qc, kc))
    golden = json.load(open(GOLDEN))["cases"][dist]
    assert oracle.fnv1a64(s) == golden["s_int32"]
    _, want_p = oracle.int_flash_pcodes(qc, qs, kc, ks, vc, vs, 128, 128)
    nflip, maxd, total = _flips(p.cpu().numpy(), want_p, _computed_tiles_mask(1024, False))
    assert maxd <= 1 and nflip <= MAX_FLIP_RATE * total, (nflip, maxd, total)


@pytest.mark.parametrize("n,d,causal,dist", [
    (4096, 128, False, "normal"),     # one C2 slice
    (4096, 128, False, "uniform"),
    (1024, 128, True, "normal"),      # causal: tiles at or below the diagonal
    (1000, 100, False, "normal"),     # ragged n, padded head dim
    (640, 64, True, "uniform"),
])
def test_s_tiles_bitwise_and_code_flips(ifa, oracle, n, d, causal, dist):
    qc, qs, kc, ks, vc, vs = _case(oracle, dist, n, d, seed=n + d)
    cfg = ifa.AttentionConfig(ifa.BlockSpec(128, 128), causal=causal)
    o, s, p = ifa.int_flash_attention_dump(_inputs(ifa, qc, qs, kc, ks, vc, vs), cfg)
    s, p = s.cpu().numpy(), p.cpu().numpy()
    mask = _computed_tiles_mask(n, causal)
    want_s = oracle.int_gemm_nt(qc, kc)
    assert np.array_equal(np.where(mask, s, 0), np.where(mask, want_s, 0))
    want_o, want_p = oracle.int_flash_pcodes(qc, qs, kc, ks, vc, vs, 128, 128,
                                             flags=2 if causal else 0)
    nflip, maxd, total = _flips(p, want_p, mask)
    assert maxd <= 1 and nflip <= MAX_FLIP_RATE * total, (nflip, maxd, total)
    # the dump instantiation's O is the product kernel's O
    fast = ifa.int_flash_attention(_inputs(ifa, qc, qs, kc, ks, vc, vs),
                                   ifa.AttentionConfig(ifa.BlockSpec(128, 128), causal=causal,
                                                       fast=True)).cpu().numpy()
    mre = float(np.abs(o.cpu().numpy().astype(np.float64) - want_o).sum() /
                np.abs(want_o).sum())
    mre_fast = float(np.abs(fast.astype(np.float64) - want_o).sum() / np.abs(want_o).sum())
    assert mre <= 1e-5 and mre_fast <= 1e-5, (mre, mre_fast)


def test_batched_slices_s_tiles(ifa, oracle):
    slices, n, d = 3, 384, 128
    cases = [_case(oracle, "normal", n, d, seed=100 + i) for i in range(slices)]
    stack = lambda i: np.stack([c[i] for c in cases])
    qc, qs, kc, ks, vc = (stack(i) for i in range(5))
    vs = np.array([c[5] for c in cases], np.float32)
    _, s, _ = ifa.int_flash_attention_dump(_inputs(ifa, qc, qs, kc, ks, vc, vs),
                                           ifa.AttentionConfig(ifa.BlockSpec(64, 128)),
                                           want_p=False)
    s = s.cpu().numpy()
    for i in range(slices):
        assert np.array_equal(s[i], oracle.int_gemm_nt(qc[i], kc[i])), i


def test_dump_rejects_other_block_sizes(ifa, oracle):
    qc, qs, kc, ks, vc, vs = _case(oracle, "normal", 512, 64)
    with pytest.raises(NotImplementedError):
        ifa.int_flash_attention_dump(_inputs(ifa, qc, qs, kc, ks, vc, vs),
                                     ifa.AttentionConfig(ifa.BlockSpec(64, 64)))

"""CPU checks of the evaluation helpers (paper_2409_16997_b200.evaluation).
The functions are device-agnostic torch code; the GPU run is in
tests/test_gpu_eval.py."""
import numpy as np
import torch


def test_reference_attention_matches_oracle_on_cpu(oracle):
    from paper_2409_16997_b200.evaluation import reference_attention
    q, k, v = oracle.slice_inputs("uniform", 96, 32, seed=5)
    want = oracle.reference_attention(q, k, v)
    got = reference_attention(*(torch.from_numpy(a) for a in (q, k, v))).numpy()
    ulps = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1


def test_causal_reference_first_row_is_first_value_row(oracle):
    from paper_2409_16997_b200.evaluation import reference_attention
    q, k, v = (torch.from_numpy(a) for a in oracle.slice_inputs("normal", 16, 8, seed=1))
    out = reference_attention(q, k, v, causal=True)
    assert torch.equal(out[0], v[0])


def test_error_accum_composes_like_the_reference(oracle):
    from paper_2409_16997_b200.evaluation import ErrorAccum, mre
    rng = np.random.default_rng(0)
    a, b = (torch.from_numpy(rng.standard_normal((8, 16)).astype(np.float32)) for _ in range(2))
    c, e = (torch.from_numpy(rng.standard_normal((8, 16)).astype(np.float32)) for _ in range(2))
    whole = ErrorAccum()
    whole.add(torch.cat([a, c]), torch.cat([b, e]))
    parts = ErrorAccum()
    p2 = ErrorAccum()
    parts.add(a, b)
    p2.add(c, e)
    parts.merge(p2)
    assert abs(parts.ratio() - whole.ratio()) < 1e-15
    assert abs(mre(a, b) - oracle.mre(a.numpy(), b.numpy())) < 1e-12


def test_outlier_injection_is_deterministic():
    from paper_2409_16997_b200.evaluation import inject_outliers
    x = np.ones((1000, 4), np.float32)
    y1 = inject_outliers(x, 0.01, 10.0, seed=7)
    y2 = inject_outliers(x, 0.01, 10.0, seed=7)
    assert np.array_equal(y1, y2)
    assert (y1[:, 0] == 10.0).sum() == 10 and (y1 == 1.0).sum() == 990 * 4

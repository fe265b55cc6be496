"""The streamed step (ifa_int8_attention_step, AttentionPlan.forward): the
quantizer runs on a few SMs concurrently with the attention kernel, which
waits per slice on a ready counter.  Its results must equal the separate
quantize + attention calls bit for bit, step after step (the counters carry
over between calls), and the quantized codes must equal the reference's."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _plans(slices, n, d, monkeypatch, **kw):
    from paper_2409_16997_b200.runtime import AttentionPlan
    monkeypatch.setenv("IFA_B200_STREAMED", "1")
    a = AttentionPlan(slices, n, d, bc=128, fast=True, **kw)
    monkeypatch.setenv("IFA_B200_STREAMED", "0")
    b = AttentionPlan(slices, n, d, bc=128, fast=True, **kw)
    return a, b


@pytest.mark.parametrize("slices,n,d,qsms", [(24, 1024, 128, "12"), (9, 512, 64, "4"),
                                             (40, 256, 128, "20"), (3, 2048, 128, "1")])
def test_streamed_step_equals_separate_calls(ifa, oracle, monkeypatch, slices, n, d, qsms):
    monkeypatch.setenv("IFA_B200_QUANT_SMS", qsms)
    streamed, plain = _plans(slices, n, d, monkeypatch)
    assert streamed.streamed and not plain.streamed
    g = torch.Generator(device="cuda").manual_seed(slices + n)
    for step in range(4):  # the ready counters carry over between steps
        q, k, v = (torch.randn(slices, n, d, device="cuda", generator=g) * (1 + step)
                   for _ in range(3))
        a = streamed.forward(q, k, v).clone()
        b = plain.forward(q, k, v)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)), step
        for name in ("qc", "kc", "vc", "sq", "sk", "sv"):
            assert torch.equal(getattr(streamed, name), getattr(plain, name)), (step, name)
        assert torch.equal(streamed.v16, plain.v16)
    streamed.check()
    # codes and scales are the reference quantizers' (oracle pinned bitwise)
    s = slices - 1
    qc, qs = oracle.quantize_per_row(q[s].cpu().numpy())
    vc, vs = oracle.quantize_per_tensor(v[s].cpu().numpy())
    assert np.array_equal(streamed.qc[s].cpu().numpy(), qc)
    assert np.array_equal(streamed.sq[s].cpu().numpy().view(np.uint32), qs.view(np.uint32))
    assert np.array_equal(streamed.vc[s].cpu().numpy(), vc)
    assert streamed.sv[s].item() == float(vs)


def test_streamed_step_reports_nonfinite(ifa, monkeypatch):
    streamed, _ = _plans(6, 256, 128, monkeypatch)
    q, k, v = (torch.randn(6, 256, 128, device="cuda") for _ in range(3))
    v[4, 7, 9] = float("inf")
    streamed.forward(q, k, v)
    with pytest.raises(ValueError, match=f"index {(4 * 256 + 7) * 128 + 9}"):
        streamed.check()
    k[1, 2, 3] = float("nan")
    streamed.forward(q, k, v)
    with pytest.raises(ValueError, match=f"index {(1 * 256 + 2) * 128 + 3}"):
        streamed.check()


def test_non_streamable_shapes_fall_back(ifa, monkeypatch):
    """Causal or ragged shapes run the separate calls inside the same entry."""
    from paper_2409_16997_b200.runtime import AttentionPlan
    monkeypatch.setenv("IFA_B200_QUANT_SMS", "12")
    for kw in ({"causal": True}, {}):
        n = 384 if kw else 300
        monkeypatch.setenv("IFA_B200_STREAMED", "1")
        p = AttentionPlan(5, n, 128, bc=128, fast=True, **kw)
        monkeypatch.setenv("IFA_B200_STREAMED", "0")
        r = AttentionPlan(5, n, 128, bc=128, fast=True, **kw)
        q, k, v = (torch.randn(5, n, 128, device="cuda") for _ in range(3))
        a = p.forward(q, k, v).clone()
        b = r.forward(q, k, v)
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)), kw

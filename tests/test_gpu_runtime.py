"""AttentionPlan (runtime.py), the executor bench.py times: same results as
the per-call API, CUDA-graph replay, and the fused fp16 V codes of the
two-Q-tile path (ifa_quantize_per_tensor_v16 / ifa_int_flash_fwd_v16)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _inputs(slices, n, d, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn((slices, n, d), generator=g, device="cuda") for _ in range(3)]


def _api(ifa, q, k, v, fast, causal=False, bc=128):
    inp = ifa.QuantizedAttentionInputs(ifa.quantize_per_row(q), ifa.quantize_per_row(k),
                                       ifa.quantize_per_tensor(v))
    return ifa.int_flash_attention(inp, ifa.AttentionConfig(ifa.BlockSpec(128, bc),
                                                            causal=causal, fast=fast))


@pytest.mark.parametrize("n,d,fast,causal", [(256, 128, True, False), (512, 64, True, False),
                                             (256, 128, False, False), (384, 128, True, True),
                                             (200, 64, True, False)])
def test_plan_matches_api_bitwise(ifa, n, d, fast, causal):
    from paper_2409_16997_b200.runtime import AttentionPlan
    q, k, v = _inputs(3, n, d, seed=n + d)
    plan = AttentionPlan(3, n, d, bc=128, causal=causal, fast=fast)
    got = plan.forward(q, k, v).clone()
    plan.check()
    want = _api(ifa, q, k, v, fast, causal)
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
    if plan.v16 is not None:  # fused fp16 copy of the V codes
        assert torch.equal(plan.v16.float(), plan.vc.float())


def test_plan_graph_replay(ifa):
    from paper_2409_16997_b200.runtime import AttentionPlan
    q, k, v = _inputs(2, 256, 128, seed=7)
    plan = AttentionPlan(2, 256, 128, bc=128, fast=True)
    want = plan.forward(q, k, v).clone()
    plan.capture(q, k, v)
    plan.out.zero_()
    plan.replay()
    torch.cuda.synchronize()
    assert torch.equal(plan.out.view(torch.int32), want.view(torch.int32))


def test_plan_launch_count(ifa):
    from paper_2409_16997_b200.runtime import AttentionPlan
    assert AttentionPlan(2, 256, 128, fast=True).launches_per_step() == 4
    assert AttentionPlan(2, 256, 128, fast=False).launches_per_step() == 4


def test_api_caller_stream_orders_readbacks(ifa):
    """A caller-supplied stream: the kernels run on it, and the host readbacks
    (non-finite check, audit) are ordered after them."""
    s = torch.cuda.Stream()
    q, k, v = _inputs(2, 256, 64, seed=3)
    k[1, 5, 7] = float("nan")
    with pytest.raises(ValueError, match=f"index {(256 + 5) * 64 + 7}"):
        ifa.quantize_per_row(k, stream=s)
    k[1, 5, 7] = 0.0
    inp = ifa.QuantizedAttentionInputs(ifa.quantize_per_row(q, stream=s),
                                       ifa.quantize_per_row(k, stream=s),
                                       ifa.quantize_per_tensor(v, stream=s))
    au = ifa.PCodeAudit()
    got = ifa.int_flash_attention(inp, ifa.AttentionConfig(ifa.BlockSpec(64, 64)), au, stream=s)
    s.synchronize()
    want = _api(ifa, q, k, v, fast=False, bc=64)
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
    assert au.rows_audited == 2 * 256 and au.max_code == 127


def test_api_rejects_bad_out_and_shapes(ifa):
    q, k, v = _inputs(1, 128, 64, seed=4)
    inp = ifa.QuantizedAttentionInputs(ifa.quantize_per_row(q), ifa.quantize_per_row(k),
                                       ifa.quantize_per_tensor(v))
    cfg = ifa.AttentionConfig(ifa.BlockSpec(64, 64))
    for bad in (torch.empty((1, 128, 32), device="cuda"),
                torch.empty((1, 128, 64), device="cuda", dtype=torch.float16),
                torch.empty((1, 64, 128), device="cuda").transpose(1, 2)):
        with pytest.raises(ValueError, match="out must be"):
            ifa.int_flash_attention(inp, cfg, out=bad)
    short = ifa.QuantizedAttentionInputs(inp.q, ifa.QuantizedRows(inp.k.values, inp.k.scales[:, :64]),
                                         inp.v)
    with pytest.raises(ValueError):
        ifa.int_flash_attention(short, cfg, validate=False)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_api_runs_on_a_non_current_device(ifa):
    """Tensors on cuda:1 while cuda:0 is current: launches go to cuda:1."""
    q, k, v = (t.to("cuda:1") for t in _inputs(1, 256, 64, seed=5))
    inp = ifa.QuantizedAttentionInputs(ifa.quantize_per_row(q), ifa.quantize_per_row(k),
                                       ifa.quantize_per_tensor(v))
    out = ifa.int_flash_attention(inp, ifa.AttentionConfig(ifa.BlockSpec(64, 64)))
    assert out.device.index == 1
    ref = _api(ifa, *(t.to("cuda:0") for t in (q, k, v)), fast=False, bc=64)
    assert torch.equal(out.cpu().view(torch.int32), ref.cpu().view(torch.int32))

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

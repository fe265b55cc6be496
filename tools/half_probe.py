"""Half-INT8 probe: tolerance numbers against the oracle and fp64, and the
C2-shape kernel time next to the full-INT8 path (one JSON line).

    python tools/half_probe.py > gpurun_out/half_probe.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2409_16997_b200 as ifa  # noqa: E402
from oracle_bindings import Oracle  # noqa: E402


def main():
    orc = Oracle()
    acc = []
    for dist, n, d in (("normal", 1024, 64), ("uniform", 1024, 128), ("normal", 4096, 128)):
        q, k, v = orc.slice_inputs(dist, n, d, seed=0)
        qq = ifa.quantize_per_row(torch.from_numpy(q).cuda())
        kq = ifa.quantize_per_row(torch.from_numpy(k).cuda())
        got = ifa.half_int8_attention(qq, kq, torch.from_numpy(v).cuda()).cpu().numpy()
        want = orc.half_int8_attention(qq.values.cpu().numpy(), qq.scales.cpu().numpy(),
                                       kq.values.cpu().numpy(), kq.scales.cpu().numpy(), v)
        exact = orc.reference_attention(q, k, v)
        acc.append({"dist": dist, "n": n, "d": d, "mre_vs_oracle": orc.mre(want, got),
                    "maxabs_vs_oracle": float(np.abs(got - want).max()),
                    "mre_fp64_gpu": orc.mre(exact, got), "mre_fp64_ref": orc.mre(exact, want)})

    slices, n, d = 128, 4096, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    x = [torch.randn((slices, n, d), generator=g, device="cuda") for _ in range(3)]
    qq, kq = ifa.quantize_per_row(x[0]), ifa.quantize_per_row(x[1])
    vq = ifa.quantize_per_tensor(x[2])
    out = torch.empty_like(x[0])
    ops = slices * 4.0 * n * n * d
    res = {}

    def timeit(name, fn, reps=10):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name] = {"ms": ms, "tops": ops / ms / 1e9}

    from paper_2409_16997_b200 import _lib
    lib = _lib.load()
    vh = x[2].half()
    sp = torch.cuda.current_stream().cuda_stream

    def half_kernel():
        _lib.check(lib.ifa_half_int8_fwd(qq.values.data_ptr(), qq.scales.data_ptr(),
                                         kq.values.data_ptr(), kq.scales.data_ptr(),
                                         vh.data_ptr(), out.data_ptr(), slices, n, d, 128, 128,
                                         0, sp))

    timeit("half_int8_kernel", half_kernel)
    timeit("half_int8_api", lambda: ifa.half_int8_attention(qq, kq, x[2], out=out))
    inp = ifa.QuantizedAttentionInputs(qq, kq, vq)
    cfg = ifa.AttentionConfig(ifa.BlockSpec(128, 128), fast=True)
    timeit("int8_fast", lambda: ifa.int_flash_attention(inp, cfg, out=out, validate=False))
    print(json.dumps({"accuracy": acc, "c2_timing": res}))


if __name__ == "__main__":
    main()

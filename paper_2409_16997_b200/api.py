"""Host-side mirror of the reference's operator interface for the hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/ifa/{quant,gemm,attention}.hpp:

=============================  ==============================================
reference                      here
=============================  ==============================================
``QuantizedRows``              :class:`QuantizedRows` (quant.hpp:17-20)
``QuantizedTensor``            :class:`QuantizedTensor` (quant.hpp:23-26)
``quantize_per_row``           :func:`quantize_per_row` (quant.hpp:30)
``quantize_per_tensor``        :func:`quantize_per_tensor` (quant.hpp:33),
                               applied per (b,h) slice as eval.cpp:101 does
``BlockSpec``                  :class:`BlockSpec` (gemm.hpp:14-19)
``AttentionConfig``            :class:`AttentionConfig` (attention.hpp:23-31)
``QuantizedAttentionInputs``   :class:`QuantizedAttentionInputs`
                               (attention.hpp:63-70, attention.cpp:213-233)
``PCodeAudit``                 :class:`PCodeAudit` (attention.hpp:75-80)
``int_flash_attention``        :func:`int_flash_attention` (attention.hpp:85-87)
``half_int8_attention``        :func:`half_int8_attention` (attention.hpp:93-96)
``fp8_e4m3_roundtrip``         :func:`fp8_quantize_per_tensor` (fp8.hpp:24-27)
``fp8_emulated_attention``     :func:`fp8_emulated_attention` (attention.hpp:98-101)
=============================  ==============================================

Tensors are ``torch`` CUDA tensors (PyTorch is only the device-memory and
stream plumbing); all arithmetic runs in libifa_b200.so.  Matrices may carry
leading batch dimensions: ``[..., n, d]`` is a batch of independent (b,h)
slices.  Exceptions: ``ValueError`` where the reference throws
``std::invalid_argument``, ``OverflowError`` for ``std::overflow_error``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _lib

K_QUANT_MAX = 127                      # quant.hpp:14
K_MAX_INT_GEMM_DEPTH = (1 << 31) // (127 * 127)  # gemm.hpp:22 (133144)
_INT64_MAX = (1 << 63) - 1


def _stream_ptr(stream: Optional[torch.cuda.Stream],
                device: Optional[torch.device] = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def _join(stream: Optional[torch.cuda.Stream], device: torch.device, *temps) -> None:
    """After launching on a caller-supplied ``stream``: keep the temporaries
    allocated on the current stream alive for ``stream`` and order the current
    stream (where host readbacks happen) after it."""
    if stream is None:
        return
    for t in temps:
        if t is not None:
            t.record_stream(stream)
    torch.cuda.current_stream(device).wait_stream(stream)


def _check_out(out: torch.Tensor, like: torch.Tensor, what: str) -> None:
    if not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or \
            out.device != like.device or tuple(out.shape) != tuple(like.shape) or \
            not out.is_contiguous():
        raise ValueError(f"{what}: out must be a contiguous float32 tensor of shape "
                         f"{tuple(like.shape)} on {like.device}")


def _require_cuda(t: torch.Tensor, dtype: torch.dtype, what: str) -> None:
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{what}: expected a torch tensor")
    if t.device.type != "cuda":
        raise ValueError(f"{what}: tensor must live on a CUDA device (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{what}: expected dtype {dtype}, got {t.dtype}")


@dataclass
class QuantizedRows:
    """Token-level quantization: one scale per row (quant.hpp:17-20)."""
    values: torch.Tensor   # int8 [..., n, d]
    scales: torch.Tensor   # f32  [..., n]


@dataclass
class QuantizedTensor:
    """Tensor-level quantization: one scale per (b,h) slice (quant.hpp:23-26)."""
    values: torch.Tensor   # int8 [..., n, d]
    scale: torch.Tensor    # f32  [...]   (0-dim for a single matrix)


@dataclass
class BlockSpec:
    """Tile sizes (gemm.hpp:14-19).  Br does not change results; Bc does."""
    Br: int = 64
    Bc: int = 64

    def validate(self) -> None:
        if self.Br < 1 or self.Bc < 1:           # gemm.cpp:16-20
            raise ValueError("BlockSpec: Br and Bc must be >= 1")


@dataclass
class AttentionConfig:
    """attention.hpp:23-31, plus the ``causal`` extension (not in the reference)."""
    blocks: BlockSpec = field(default_factory=BlockSpec)
    apply_sqrt_d_scaling: bool = False
    causal: bool = False
    # tolerance mode (IFA_FLAG_FAST): O within the stated tolerance instead of
    # bitwise; codes, scales and S stay exact
    fast: bool = False

    def validate(self) -> None:
        self.blocks.validate()


@dataclass
class PCodeAudit:
    """attention.hpp:75-80."""
    min_code: int = 127
    max_code: int = 0
    row_max_block_hits_127: bool = True
    rows_audited: int = 0


@dataclass
class QuantizedAttentionInputs:
    q: QuantizedRows
    k: QuantizedRows
    v: QuantizedTensor

    def validate(self) -> None:
        """attention.cpp:213-233 (the sV check reads the scales back to the host)."""
        qv = self.q.values
        if qv.dim() < 2 or qv.shape[-2] < 1 or qv.shape[-1] < 1:
            raise ValueError("quantized attention inputs: empty q")
        n, d = qv.shape[-2], qv.shape[-1]
        for name, t in (("k", self.k.values), ("v", self.v.values)):
            if tuple(t.shape) != tuple(qv.shape):
                raise ValueError(
                    f"quantized attention inputs: q, k, v must all be {n}x{d} "
                    f"(got {name} {tuple(t.shape)})")
        for name, s in (("q", self.q.scales), ("k", self.k.scales)):
            if tuple(s.shape) != tuple(qv.shape[:-1]):
                raise ValueError(
                    f"quantized attention inputs: scale vectors must have length {n}")
        sv = self.v.scale
        if tuple(sv.shape) != tuple(qv.shape[:-2]):
            raise ValueError("quantized attention inputs: one v scale per slice expected")
        bad = ~(torch.isfinite(sv) & (sv >= 0))
        if bool(bad.any()):
            raise ValueError("quantized attention inputs: bad v scale")


def quantize_per_row(x: torch.Tensor, *, check_finite: bool = True,
                     stream: Optional[torch.cuda.Stream] = None) -> QuantizedRows:
    """codes = round_half_away(x / scale_row), scale_row = max|x_row| / 127 (quant.cpp:44-57).

    ``check_finite`` mirrors quant.cpp:14-22 (reads one int64 back).
    """
    _require_cuda(x, torch.float32, "quantize_per_row")
    if x.dim() < 2:
        raise ValueError("quantize_per_row: expected a matrix [..., rows, cols]")
    x = x.contiguous()
    cols = x.shape[-1]
    rows = x.numel() // cols if cols else 0
    codes = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    scales = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    bad = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=x.device) if check_finite \
        else None
    lib = _lib.load()
    with torch.cuda.device(x.device):
        _lib.check(lib.ifa_quantize_per_row(x.data_ptr(), rows, cols, codes.data_ptr(),
                                            scales.data_ptr(),
                                            bad.data_ptr() if bad is not None else None,
                                            _stream_ptr(stream, x.device)))
    _join(stream, x.device, bad)
    if bad is not None:
        idx = int(bad.item())
        if idx != _INT64_MAX:
            raise ValueError(f"quantize_per_row: non-finite input at index {idx}")
    return QuantizedRows(codes, scales)


def quantize_per_tensor(x: torch.Tensor, *, check_finite: bool = True,
                        stream: Optional[torch.cuda.Stream] = None) -> QuantizedTensor:
    """One scale max|x_slice| / 127 per trailing [rows, cols] matrix (quant.cpp:59-69)."""
    _require_cuda(x, torch.float32, "quantize_per_tensor")
    if x.dim() < 2:
        raise ValueError("quantize_per_tensor: expected a matrix [..., rows, cols]")
    x = x.contiguous()
    rows, cols = x.shape[-2], x.shape[-1]
    slices = x.numel() // (rows * cols) if rows * cols else math.prod(x.shape[:-2])
    codes = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    scale = torch.empty(x.shape[:-2], dtype=torch.float32, device=x.device)
    ws = torch.empty(max(slices, 1), dtype=torch.int32, device=x.device)
    bad = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=x.device) if check_finite \
        else None
    lib = _lib.load()
    with torch.cuda.device(x.device):
        _lib.check(lib.ifa_quantize_per_tensor(x.data_ptr(), slices, rows, cols,
                                               codes.data_ptr(), scale.data_ptr(), ws.data_ptr(),
                                               bad.data_ptr() if bad is not None else None,
                                               _stream_ptr(stream, x.device)))
    _join(stream, x.device, bad, ws)
    if bad is not None:
        idx = int(bad.item())
        if idx != _INT64_MAX:
            raise ValueError(f"quantize_per_tensor: non-finite input at index {idx}")
    return QuantizedTensor(codes, scale)


def int_flash_attention(inputs: QuantizedAttentionInputs,
                        cfg: Optional[AttentionConfig] = None,
                        audit: Optional[PCodeAudit] = None, *,
                        out: Optional[torch.Tensor] = None,
                        validate: bool = True,
                        stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Full-INT8 tiled attention (attention.hpp:82-87) on the GPU.

    Returns f32 O with the shape of ``inputs.q.values``.  ``audit`` (if given)
    is filled like the reference's PCodeAudit (one host readback).
    ``validate=False`` skips the host-side sV check (no device sync).
    """
    cfg = cfg or AttentionConfig()
    qv, kv, vv = inputs.q.values, inputs.k.values, inputs.v.values
    for name, t in (("q", qv), ("k", kv), ("v", vv)):
        _require_cuda(t, torch.int8, f"int_flash_attention: {name}")
    if validate:
        inputs.validate()
    else:
        _check_shapes(inputs)
    cfg.validate()
    n, d = qv.shape[-2], qv.shape[-1]
    slices = qv.numel() // (n * d)
    q, k, v = qv.contiguous(), kv.contiguous(), vv.contiguous()
    sq = inputs.q.scales.contiguous()
    sk = inputs.k.scales.contiguous()
    sv = inputs.v.scale.contiguous().reshape(-1)
    if out is None:
        out = torch.empty(qv.shape, dtype=torch.float32, device=qv.device)
    else:
        _check_out(out, qv, "int_flash_attention")
    flags = (_lib.FLAG_SQRT_D if cfg.apply_sqrt_d_scaling else 0) | \
        (_lib.FLAG_CAUSAL if cfg.causal else 0) | (_lib.FLAG_FAST if cfg.fast else 0)
    lib = _lib.load()
    au = None
    with torch.cuda.device(qv.device):
        sp = _stream_ptr(stream, qv.device)
        if audit is not None:
            au = torch.empty(3, dtype=torch.int64, device=qv.device)  # 24 bytes
            _lib.check(lib.ifa_audit_init(au.data_ptr(), sp))
        _lib.check(lib.ifa_int_flash_fwd(q.data_ptr(), sq.data_ptr(), k.data_ptr(),
                                         sk.data_ptr(), v.data_ptr(), sv.data_ptr(),
                                         out.data_ptr(), slices, n, d, cfg.blocks.Br,
                                         cfg.blocks.Bc, flags,
                                         au.data_ptr() if au is not None else None, sp))
    _join(stream, qv.device, au)
    if au is not None:
        raw = au.cpu().numpy()
        w = raw[:2].view("int32")
        audit.min_code = int(w[0])
        audit.max_code = int(w[1])
        audit.row_max_block_hits_127 = bool(w[2])
        audit.rows_audited = int(raw[2])
    return out


def _check_shapes(inputs: QuantizedAttentionInputs) -> None:
    """The cheap (no device sync) part of QuantizedAttentionInputs.validate
    plus dtypes: what the kernels need to stay in bounds."""
    qv = inputs.q.values
    if qv.dim() < 2 or qv.shape[-2] < 1 or qv.shape[-1] < 1:
        raise ValueError("quantized attention inputs: empty q")
    for name, t in (("k", inputs.k.values), ("v", inputs.v.values)):
        if tuple(t.shape) != tuple(qv.shape):
            raise ValueError(f"quantized attention inputs: q, k, v must all be "
                             f"{qv.shape[-2]}x{qv.shape[-1]} (got {name} {tuple(t.shape)})")
    for name, sc, shape in (("q", inputs.q.scales, qv.shape[:-1]),
                            ("k", inputs.k.scales, qv.shape[:-1]),
                            ("v", inputs.v.scale, qv.shape[:-2])):
        _require_cuda(sc, torch.float32, f"quantized attention inputs: {name} scales")
        if tuple(sc.shape) != tuple(shape):
            raise ValueError(f"quantized attention inputs: bad {name} scale shape "
                             f"{tuple(sc.shape)}")
        if sc.device != qv.device:
            raise ValueError("quantized attention inputs: tensors on different devices")


def int_flash_attention_dump(inputs: QuantizedAttentionInputs,
                             cfg: Optional[AttentionConfig] = None, *,
                             want_s: bool = True, want_p: bool = True,
                             stream: Optional[torch.cuda.Stream] = None):
    """Tolerance-mode forward that also returns what the tensor core computed:
    ``(O, S, P)`` with S int32 ``[..., n, n]`` = Q.K^T read back from the
    kind::i8 TMEM accumulator (the reference's int_gemm_nt,
    attention.cpp:275-276 / gemm.cpp:32-46) and P uint8 ``[..., n, n]`` the
    weight codes fed to P.V (attention.cpp:299-312); either may be None.
    Needs Bc = 128 (the kernel's KV tile) or Bc >= n <= 128.  With ``causal``
    only KV tiles at or below the diagonal are written (others stay 0)."""
    cfg = cfg or AttentionConfig()
    qv = inputs.q.values
    for name, t in (("q", qv), ("k", inputs.k.values), ("v", inputs.v.values)):
        _require_cuda(t, torch.int8, f"int_flash_attention: {name}")
    inputs.validate()
    cfg.validate()
    n, d = qv.shape[-2], qv.shape[-1]
    slices = qv.numel() // (n * d)
    lead = tuple(qv.shape[:-2])
    out = torch.empty(qv.shape, dtype=torch.float32, device=qv.device)
    s_out = torch.zeros(lead + (n, n), dtype=torch.int32, device=qv.device) if want_s else None
    p_out = torch.zeros(lead + (n, n), dtype=torch.uint8, device=qv.device) if want_p else None
    flags = _lib.FLAG_FAST | _lib.FLAG_DUMP_S | \
        (_lib.FLAG_SQRT_D if cfg.apply_sqrt_d_scaling else 0) | \
        (_lib.FLAG_CAUSAL if cfg.causal else 0)
    lib = _lib.load()
    with torch.cuda.device(qv.device):
        _lib.check(lib.ifa_int_flash_fwd_dump(
            inputs.q.values.contiguous().data_ptr(), inputs.q.scales.contiguous().data_ptr(),
            inputs.k.values.contiguous().data_ptr(), inputs.k.scales.contiguous().data_ptr(),
            inputs.v.values.contiguous().data_ptr(),
            inputs.v.scale.contiguous().reshape(-1).data_ptr(), out.data_ptr(), slices, n, d,
            cfg.blocks.Br, cfg.blocks.Bc, flags,
            s_out.data_ptr() if s_out is not None else None,
            p_out.data_ptr() if p_out is not None else None, _stream_ptr(stream, qv.device)))
    _join(stream, qv.device)
    return out, s_out, p_out


def half_int8_attention(q: QuantizedRows, k: QuantizedRows, v: torch.Tensor,
                        cfg: Optional[AttentionConfig] = None, *,
                        out: Optional[torch.Tensor] = None,
                        stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Half-INT8 attention (attention.hpp:93-96, attention.cpp:359-399) on the GPU.

    int8 Q/K with per-row scales, float V and float attention weights.  V
    (f32 ``[..., n, d]``) is converted to fp16 on the device and the weights
    go to the tensor core as fp16 with fp32 accumulation: O agrees with the
    reference within the tolerance tests/test_gpu_half.py states, not
    bitwise.  ``cfg.blocks`` is validated (it changes only float rounding
    order in the reference); ``causal``/``fast`` are not part of this path.
    """
    cfg = cfg or AttentionConfig()
    qv, kv = q.values, k.values
    _require_cuda(qv, torch.int8, "half_int8_attention: q")
    _require_cuda(kv, torch.int8, "half_int8_attention: k")
    _require_cuda(v, torch.float32, "half_int8_attention: v")
    if qv.dim() < 2 or qv.shape[-2] < 1 or qv.shape[-1] < 1 or v.shape[-1] < 1:
        raise ValueError("half_int8_attention: empty input")       # attention.cpp:374-376
    if kv.shape[-1] != qv.shape[-1]:
        raise ValueError("half_int8_attention: q/k head dims differ")  # :364-366
    if kv.shape[-2] != v.shape[-2]:
        raise ValueError("half_int8_attention: k/v row counts differ")  # :367-369
    if tuple(q.scales.shape) != tuple(qv.shape[:-1]) or \
            tuple(k.scales.shape) != tuple(kv.shape[:-1]):
        raise ValueError("half_int8_attention: scale length mismatch")  # :370-373
    if tuple(kv.shape) != tuple(qv.shape) or tuple(v.shape) != tuple(qv.shape):
        raise NotImplementedError(
            "half_int8_attention: the sm_100a kernel takes q, k, v of one shape [..., n, d]")
    cfg.validate()
    if cfg.causal or cfg.fast:
        raise NotImplementedError("half_int8_attention: causal/fast are not part of this path")
    n, d = qv.shape[-2], qv.shape[-1]
    slices = qv.numel() // (n * d)
    qc, kc = qv.contiguous(), kv.contiguous()
    sq, sk = q.scales.contiguous(), k.scales.contiguous()
    vc = v.contiguous()
    # the kernel feeds V to the tensor core as fp16: |V| beyond the fp16
    # range (65504) would become inf, so refuse it instead of returning inf/NaN
    if vc.numel() and float(vc.abs().max()) > 65504.0:
        raise ValueError("half_int8_attention: |v| exceeds the fp16 range (65504) of the "
                         "sm_100a kernel")
    vh = torch.empty(v.shape, dtype=torch.float16, device=v.device)
    if out is None:
        out = torch.empty(qv.shape, dtype=torch.float32, device=qv.device)
    else:
        _check_out(out, qv, "half_int8_attention")
    lib = _lib.load()
    with torch.cuda.device(qv.device):
        sp = _stream_ptr(stream, qv.device)
        _lib.check(lib.ifa_convert_f16(vc.data_ptr(), vc.numel(), vh.data_ptr(), sp))
        _lib.check(lib.ifa_half_int8_fwd(qc.data_ptr(), sq.data_ptr(), kc.data_ptr(),
                                         sk.data_ptr(), vh.data_ptr(), out.data_ptr(), slices,
                                         n, d, cfg.blocks.Br, cfg.blocks.Bc,
                                         _lib.FLAG_SQRT_D if cfg.apply_sqrt_d_scaling else 0,
                                         sp))
    _join(stream, qv.device, vh)
    return out


@dataclass
class Fp8Tensor:
    """e4m3 codes of a fp8_e4m3_roundtrip per (b,h) slice (fp8.cpp:78-97):
    restored = decode(codes) / scale."""
    codes: torch.Tensor     # uint8 [..., n, d] (e4m3 bit patterns)
    scale: torch.Tensor     # f32 [...] (448 / max|x| per slice; 0 for all-zero)
    decoded: torch.Tensor   # fp16 [..., n, d] = decode(codes), exact


def fp8_quantize_per_tensor(x: torch.Tensor, *, check_finite: bool = True,
                            stream: Optional[torch.cuda.Stream] = None) -> Fp8Tensor:
    """fp8_e4m3_roundtrip's quantization of each trailing [rows, cols] matrix
    on the GPU; codes bitwise equal to the reference's e4m3_encode."""
    _require_cuda(x, torch.float32, "fp8_e4m3_roundtrip")
    if x.dim() < 2:
        raise ValueError("fp8_e4m3_roundtrip: expected a matrix [..., rows, cols]")
    x = x.contiguous()
    rows, cols = x.shape[-2], x.shape[-1]
    slices = math.prod(x.shape[:-2]) if x.dim() > 2 else 1
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    dec = torch.empty(x.shape, dtype=torch.float16, device=x.device)
    scale = torch.empty(x.shape[:-2], dtype=torch.float32, device=x.device)
    ws = torch.empty(max(slices, 1), dtype=torch.int32, device=x.device)
    bad = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=x.device) if check_finite \
        else None
    lib = _lib.load()
    with torch.cuda.device(x.device):
        _lib.check(lib.ifa_fp8_quantize_per_tensor(x.data_ptr(), slices, rows, cols,
                                                   codes.data_ptr(), dec.data_ptr(),
                                                   scale.data_ptr(), ws.data_ptr(),
                                                   bad.data_ptr() if bad is not None else None,
                                                   _stream_ptr(stream, x.device)))
    _join(stream, x.device, bad, ws)
    if bad is not None and int(bad.item()) != _INT64_MAX:
        raise ValueError("fp8_e4m3_roundtrip: non-finite input")  # fp8.cpp:82-84
    return Fp8Tensor(codes, scale, dec)


def fp8_emulated_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                           cfg: Optional[AttentionConfig] = None, *,
                           out: Optional[torch.Tensor] = None,
                           stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """fp8_emulated_attention (attention.cpp:401-407) on the GPU, natively in
    FP8: e4m3 Q/K on the tensor core (tcgen05 kind::f8f6f4), float softmax,
    P (fp16) . V (decoded e4m3).  f32 [..., n, d] in, f32 O out; within the
    tolerance tests/test_gpu_fp8.py states of the reference."""
    cfg = cfg or AttentionConfig()
    for name, t in (("q", q), ("k", k), ("v", v)):
        _require_cuda(t, torch.float32, f"fp8_emulated_attention: {name}")
    if q.dim() < 2 or q.shape[-2] < 1 or q.shape[-1] < 1:
        raise ValueError("fp8_emulated_attention: empty input")
    if tuple(k.shape) != tuple(q.shape) or tuple(v.shape) != tuple(q.shape):
        raise NotImplementedError(
            "fp8_emulated_attention: the sm_100a kernel takes q, k, v of one shape [..., n, d]")
    cfg.validate()
    if cfg.causal or cfg.fast:
        raise NotImplementedError("fp8_emulated_attention: causal/fast are not part of this path")
    n, d = q.shape[-2], q.shape[-1]
    slices = q.numel() // (n * d)
    q8, k8, v8 = (fp8_quantize_per_tensor(t, stream=stream) for t in (q, k, v))
    if out is None:
        out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    else:
        _check_out(out, q, "fp8_emulated_attention")
    lib = _lib.load()
    with torch.cuda.device(q.device):
        _lib.check(lib.ifa_fp8_attention_fwd(q8.codes.data_ptr(), q8.scale.data_ptr(),
                                             k8.codes.data_ptr(), k8.scale.data_ptr(),
                                             v8.decoded.data_ptr(), v8.scale.data_ptr(),
                                             out.data_ptr(), slices, n, d, cfg.blocks.Br,
                                             cfg.blocks.Bc,
                                             _lib.FLAG_SQRT_D if cfg.apply_sqrt_d_scaling
                                             else 0, _stream_ptr(stream, q.device)))
    _join(stream, q.device, q8.codes, q8.scale, q8.decoded, k8.codes, k8.scale, k8.decoded,
          v8.codes, v8.scale, v8.decoded)
    return out


def version() -> str:
    return _lib.load().ifa_version().decode()

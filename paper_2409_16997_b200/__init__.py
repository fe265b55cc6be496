"""B200-native INT-FlashAttention forward (arXiv 2409.16997 hot path).

Per-token INT8 quantization of Q/K, per-slice tensor-level INT8
quantization of V, and the fused full-INT8 flash-attention forward, as
hand-written sm_100a kernels (TMA + tcgen05.mma kind::i8 + TMEM) behind the
C-ABI in include/ifa_b200.h.  See DESIGN.md.
"""
from .api import (  # noqa: F401
    AttentionConfig,
    BlockSpec,
    PCodeAudit,
    QuantizedAttentionInputs,
    QuantizedRows,
    QuantizedTensor,
    Fp8Tensor,
    fp8_emulated_attention,
    fp8_quantize_per_tensor,
    half_int8_attention,
    int_flash_attention,
    int_flash_attention_dump,
    quantize_per_row,
    quantize_per_tensor,
    version,
)
from ._lib import NativeLibraryError  # noqa: F401

__all__ = [
    "AttentionConfig", "BlockSpec", "PCodeAudit", "QuantizedAttentionInputs",
    "QuantizedRows", "QuantizedTensor", "Fp8Tensor", "fp8_emulated_attention",
    "fp8_quantize_per_tensor", "half_int8_attention", "int_flash_attention", "int_flash_attention_dump", "quantize_per_row",
    "quantize_per_tensor", "version", "NativeLibraryError",
]

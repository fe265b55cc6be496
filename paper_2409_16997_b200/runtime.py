"""Pre-planned execution of the whole hot path (quantize Q, K, V + INT8
flash attention) for a fixed [slices, n, d] shape.

``AttentionPlan`` owns every device buffer the path needs (codes, scales,
V-absmax workspace, non-finite detector, output) so a step is four C-ABI
calls on one stream with no allocation and no host synchronisation; the
reference's non-finite rejection (quant.cpp:14-22) is folded into a device
word that ``check()`` reads once.  ``capture()`` records a step into a CUDA
graph for launch-bound (small) shapes.  This is the executor ``bench.py``
and multi-GPU runs use; the per-call API in ``api.py`` is the drop-in
mirror of the reference functions.
"""
from __future__ import annotations

import os
from typing import Optional

import torch

from . import _lib

_INT64_MAX = (1 << 63) - 1


class AttentionPlan:
    def __init__(self, slices: int, n: int, d: int, *, bc: int = 128, br: int = 128,
                 causal: bool = False, sqrt_d: bool = False, fast: bool = False,
                 device: Optional[torch.device] = None):
        if slices < 1 or n < 1 or d < 1:
            raise ValueError("AttentionPlan: slices, n and d must be >= 1")
        if bc < 1 or br < 1:
            raise ValueError("BlockSpec: Br and Bc must be >= 1")
        self.lib = _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.slices, self.n, self.d, self.bc, self.br = slices, n, d, bc, br
        self.flags = (_lib.FLAG_CAUSAL if causal else 0) | (_lib.FLAG_SQRT_D if sqrt_d else 0) | \
            (_lib.FLAG_FAST if fast else 0)
        shape = (slices, n, d)
        self.qc = torch.empty(shape, dtype=torch.int8, device=dev)
        self.kc = torch.empty(shape, dtype=torch.int8, device=dev)
        self.vc = torch.empty(shape, dtype=torch.int8, device=dev)
        self.sq = torch.empty((slices, n), dtype=torch.float32, device=dev)
        self.sk = torch.empty((slices, n), dtype=torch.float32, device=dev)
        self.sv = torch.empty((slices,), dtype=torch.float32, device=dev)
        self.out = torch.empty(shape, dtype=torch.float32, device=dev)
        self.ws = torch.empty((slices,), dtype=torch.int32, device=dev)
        self.bad = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=dev)
        # fp16 V codes for the two-Q-tile kernel, written by the V quantizer
        self.v16 = torch.empty(shape, dtype=torch.float16, device=dev) \
            if self.uses_pp_kernel() and d in (64, 128) and n % 128 == 0 else None
        # V (two passes + a cluster sync per slice) runs on a side stream next to
        # the single-pass Q/K row kernels, so HBM stays busy through V's syncs
        # streamed step (ifa_int8_attention_step): per-slice ready counters
        self._sync = torch.zeros((2 * slices,), dtype=torch.int32, device=dev) \
            if self.v16 is not None else None
        self._epoch = 0
        # off by default: measured slower than quantize-then-attention on C2 and
        # C5; IFA_B200_STREAMED=1 selects it
        self.streamed = self.v16 is not None and os.environ.get("IFA_B200_STREAMED", "0") == "1"
        self._side = torch.cuda.Stream(dev)
        self._fork = torch.cuda.Event()
        self._join = torch.cuda.Event()
        self.graph: Optional[torch.cuda.CUDAGraph] = None
        self._graph_io = None

    # ------------------------------------------------------------------
    def quantize(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                 stream: Optional[torch.cuda.Stream] = None) -> None:
        main = stream or torch.cuda.current_stream(self.device)
        s = int(main.cuda_stream)
        L, rows, d = self.lib, self.slices * self.n, self.d
        bad = self.bad.data_ptr()
        self._fork.record(main)
        self._side.wait_event(self._fork)
        sv = int(self._side.cuda_stream)
        if self.v16 is not None:
            _lib.check(L.ifa_quantize_per_tensor_v16(v.data_ptr(), self.slices, self.n, d,
                                                     self.vc.data_ptr(), self.v16.data_ptr(),
                                                     self.sv.data_ptr(), self.ws.data_ptr(),
                                                     bad, sv))
        else:
            _lib.check(L.ifa_quantize_per_tensor(v.data_ptr(), self.slices, self.n, d,
                                                 self.vc.data_ptr(), self.sv.data_ptr(),
                                                 self.ws.data_ptr(), bad, sv))
        _lib.check(L.ifa_quantize_per_row(q.data_ptr(), rows, d, self.qc.data_ptr(),
                                          self.sq.data_ptr(), bad, s))
        _lib.check(L.ifa_quantize_per_row(k.data_ptr(), rows, d, self.kc.data_ptr(),
                                          self.sk.data_ptr(), bad, s))
        self._join.record(self._side)
        main.wait_event(self._join)

    def attention(self, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        s = int((stream or torch.cuda.current_stream(self.device)).cuda_stream)
        if self.v16 is not None:
            _lib.check(self.lib.ifa_int_flash_fwd_v16(
                self.qc.data_ptr(), self.sq.data_ptr(), self.kc.data_ptr(), self.sk.data_ptr(),
                self.vc.data_ptr(), self.v16.data_ptr(), self.sv.data_ptr(), self.out.data_ptr(),
                self.slices, self.n, self.d, self.br, self.bc, self.flags, s))
            return self.out
        _lib.check(self.lib.ifa_int_flash_fwd(
            self.qc.data_ptr(), self.sq.data_ptr(), self.kc.data_ptr(), self.sk.data_ptr(),
            self.vc.data_ptr(), self.sv.data_ptr(), self.out.data_ptr(), self.slices, self.n,
            self.d, self.br, self.bc, self.flags, None, s))
        return self.out

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """quantize_per_row(Q), quantize_per_row(K), quantize_per_tensor(V) per
        slice, then int_flash_attention; inputs f32 [slices, n, d] on device."""
        for t in (q, k, v):
            if t.dtype != torch.float32 or not t.is_contiguous() or \
                    tuple(t.shape) != (self.slices, self.n, self.d) or t.device != self.device:
                raise ValueError("AttentionPlan.forward: expected contiguous f32 "
                                 f"{(self.slices, self.n, self.d)} tensors on {self.device}")
        if self.streamed:
            return self.step(q, k, v, stream)
        self.quantize(q, k, v, stream)
        return self.attention(stream)

    def step(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """The whole step as one ifa_int8_attention_step call: the quantizer
        runs on a few SMs next to the attention kernel, which waits per slice
        (same results as quantize() + attention())."""
        assert self._sync is not None, "step() needs the fp16-V (two-Q-tile) configuration"
        s = int((stream or torch.cuda.current_stream(self.device)).cuda_stream)
        self._epoch += 1
        if self._epoch >= 1 << 31:  # the ready words hold the epoch
            self._sync.zero_()
            self._epoch = 1
        _lib.check(self.lib.ifa_int8_attention_step(
            q.data_ptr(), k.data_ptr(), v.data_ptr(), self.qc.data_ptr(), self.sq.data_ptr(),
            self.kc.data_ptr(), self.sk.data_ptr(), self.vc.data_ptr(), self.sv.data_ptr(),
            self.v16.data_ptr(), self.out.data_ptr(), self.bad.data_ptr(),
            self._sync.data_ptr(), self._epoch, self.slices, self.n, self.d, self.br, self.bc,
            self.flags, s))
        return self.out

    def uses_pp_kernel(self) -> bool:
        """True when ifa_int_flash_fwd takes the two-Q-tile tolerance kernel
        (csrc/attn_pp.cu: fast mode, Bc = 128),
        which first converts the V codes to fp16 (one extra launch)."""
        bc = min(self.bc, self.n)
        blocks = bc == 128 or (bc == self.n and self.n <= 128)
        return bool(self.flags & _lib.FLAG_FAST) and blocks and self.d <= 128 and \
            os.environ.get("IFA_B200_NO_PP", "") != "1"

    def launches_per_step(self) -> int:
        """Kernels one forward() launches (quantize: Q rows, K rows, fused V
        slices -- or absmax + quantize + a memset on shapes the fused V
        kernel does not take; attention: one persistent kernel, plus the V
        fp16 conversion on the two-Q-tile path)."""
        if self.streamed:
            return 5  # first slices: Q rows, K rows, V; stream quantizer; attention
        elems = self.n * self.d
        v_fused = elems % 16 == 0 and self.d % 4 == 0
        pp = self.uses_pp_kernel()
        conv = pp and (self.v16 is None or not v_fused)  # separate int8 -> fp16 pass
        return 2 + (1 if v_fused else 3) + 1 + (1 if conv else 0)

    def check(self) -> None:
        """Raise like the reference if any quantized input was non-finite."""
        idx = int(self.bad.item())
        if idx != _INT64_MAX:
            self.bad.fill_(_INT64_MAX)
            raise ValueError(f"quantize: non-finite input at index {idx}")

    # ------------------------------------------------------------------
    def capture(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> None:
        """Record forward(q, k, v) into a CUDA graph (replay with ``replay()``)."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        # a graph replays fixed kernel arguments, so the streamed step (whose
        # epoch advances every call) is not captured: quantize + attention
        with torch.cuda.stream(s):
            self.quantize(q, k, v, s)  # warm-up outside the graph (lazy init)
            self.attention(s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.quantize(q, k, v)
            self.attention()
        self.graph = g
        self._graph_io = (q, k, v)

    def replay(self) -> torch.Tensor:
        assert self.graph is not None, "capture() first"
        self.graph.replay()
        return self.out

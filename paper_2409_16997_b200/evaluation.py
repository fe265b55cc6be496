"""GPU evaluation side of the path: the fp64
ground-truth attention and the normalized-L1 error the reference reports.

- :func:`reference_attention` restates ``ifa::reference_attention``
  (/root/reference/proj/src/attention.cpp:151-192): scores, softmax and the
  weighted sum in float64, output rounded once to float32.  It runs as
  float64 GEMMs on the device in row blocks, so an N=16k slice takes
  milliseconds instead of the reference's ~35 s per slice on one core.
- :class:`ErrorAccum` restates ``ErrorAccum`` (eval.cpp:55-75): numerator and
  denominator of the normalized L1 ratio kept separately, so several
  matrices (the (b,h) slices of one seed) share one quotient and partial sums
  from several GPUs compose exactly (sum the pairs, then divide).
- :func:`inject_outliers` is this build's outlier-token definition for the C4
  sweep (the reference has none): ``round(frac * n)``
  distinct rows chosen by a seeded partial Fisher-Yates, scaled by ``factor``.

This module is evaluation tooling around the hot path.  The product kernels
are in csrc/ and run through api.py / runtime.py.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch


def reference_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *,
                        sqrt_d: bool = False, causal: bool = False,
                        row_block: int = 2048) -> torch.Tensor:
    """Untiled softmax(Q K^T [/ sqrt(d)]) V in float64, rounded to float32.

    ``q, k, v``: float32 ``[..., n, d]`` CUDA tensors (one or more slices).
    ``causal`` (extension, not in the reference): row i sees keys j <= i.
    """
    if q.shape != k.shape or q.shape[:-1] != v.shape[:-1]:
        raise ValueError("reference_attention: q, k, v shapes disagree")
    n, d = q.shape[-2], q.shape[-1]
    scale = 1.0 / float(np.sqrt(d)) if sqrt_d else 1.0
    q64 = q.to(torch.float64)
    k64 = k.to(torch.float64)
    v64 = v.to(torch.float64)
    out = torch.empty(v.shape, dtype=torch.float32, device=v.device)
    for r0 in range(0, n, row_block):
        r1 = min(n, r0 + row_block)
        s = torch.matmul(q64[..., r0:r1, :], k64.transpose(-1, -2)) * scale
        if causal:
            rows = torch.arange(r0, r1, device=q.device).unsqueeze(1)
            cols = torch.arange(n, device=q.device).unsqueeze(0)
            s = s.masked_fill(cols > rows, float("-inf"))
        s = s - s.amax(dim=-1, keepdim=True)
        w = torch.exp(s)
        l = w.sum(dim=-1, keepdim=True)
        out[..., r0:r1, :] = (torch.matmul(w, v64) / l).to(torch.float32)
    return out


class ErrorAccum:
    """Normalized L1 error, numerator and denominator kept apart (eval.cpp:55-75)."""

    def __init__(self):
        self.num = 0.0
        self.den = 0.0

    def add(self, reference: torch.Tensor, candidate: torch.Tensor) -> None:
        if reference.shape != candidate.shape:
            raise ValueError("mre: shape mismatch")
        r = reference.to(torch.float64)
        c = candidate.to(torch.float64)
        self.num += float((c - r).abs().sum())
        self.den += float(r.abs().sum())

    def merge(self, other: "ErrorAccum") -> None:
        self.num += other.num
        self.den += other.den

    def ratio(self) -> float:
        if self.den == 0.0:
            raise ZeroDivisionError("mre: reference is all zero")  # eval.cpp:70-72
        return self.num / self.den


def mre(reference: torch.Tensor, candidate: torch.Tensor) -> float:
    """eval.cpp:249-253 (ifa::mre)."""
    acc = ErrorAccum()
    acc.add(reference, candidate)
    return acc.ratio()


def inject_outliers(x: np.ndarray, frac: float, factor: float, seed: int,
                    rng: Optional[np.random.Generator] = None) -> np.ndarray:
    """Scale ``round(frac * n)`` distinct rows of ``x`` (n x d) by ``factor``.

    Rows come from a partial Fisher-Yates shuffle driven by
    ``numpy.random.Generator(PCG64(seed))``.  Returns a copy.
    """
    n = x.shape[0]
    count = int(round(frac * n))
    rng = rng or np.random.Generator(np.random.PCG64(seed))
    idx = np.arange(n)
    for i in range(count):
        j = int(rng.integers(i, n))
        idx[i], idx[j] = idx[j], idx[i]
    out = np.array(x, dtype=np.float32, copy=True)
    out[idx[:count]] *= np.float32(factor)
    return out

"""Attention math API of the reference (tierkv/attention.py) on the B200.

Same names, argument meaning, dtype contract and ContractError behaviour as
attention.py:30-199; the arithmetic runs in libhgca_b200.so. Inputs may be
numpy arrays (results come back as numpy, so this is a drop-in for the
reference module) or torch tensors (results stay on the device).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dev import DTYPE_CODE, as_device, back, device, stream_handle
from .errors import ContractError

__all__ = ["HeadShape", "AttentionResult", "attend", "attend_indexed", "merge_states", "logsumexp"]


@dataclass(frozen=True)
class HeadShape:
    """attention.py:40-60: head count, head dimension, score scale (1/sqrt(d))."""

    num_heads: int
    head_dim: int
    scale: float | None = None

    def __post_init__(self):
        if self.num_heads < 1:
            raise ContractError(f"num_heads must be >= 1, got {self.num_heads}")
        if self.head_dim < 1:
            raise ContractError(f"head_dim must be >= 1, got {self.head_dim}")
        if self.scale is None:
            object.__setattr__(self, "scale", 1.0 / math.sqrt(self.head_dim))
        if self.scale <= 0:
            raise ContractError(f"scale must be > 0, got {self.scale}")


@dataclass
class AttentionResult:
    """attention.py:63-75: output [..., nq, d], lse [..., nq] float64, weights."""

    output: object
    lse: object
    weights: object = None


def _working(x, name):
    """attention.py:78-84: non-float32/64 inputs become float64; 2-D or 3-D."""
    t, is_np = as_device(x)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    if t.dim() not in (2, 3):
        raise ContractError(f"{name} must be 2-D or 3-D, got shape {tuple(t.shape)}")
    return t.contiguous(), is_np


def _promote(*ts):
    dt = torch.float64 if any(t.dtype == torch.float64 for t in ts) else torch.float32
    return [t.to(dt) for t in ts]


def attend(q, k, v, shape: HeadShape, keep_weights: bool = False) -> AttentionResult:
    """Dense attention (attention.py:87-124) through hgca_attend_dense."""
    (q, np_q), (k, _), (v, _) = _working(q, "q"), _working(k, "k"), _working(v, "v")
    if not (q.dim() == k.dim() == v.dim()):
        raise ContractError("q, k, v must all be 2-D or all be 3-D")
    single = q.dim() == 2
    if single:
        q, k, v = q[None], k[None], v[None]
    if q.shape[0] != shape.num_heads and not (single and shape.num_heads == 1):
        raise ContractError(f"expected {shape.num_heads} heads, got {q.shape[0]}")
    if q.shape[2] != shape.head_dim or k.shape[2] != shape.head_dim:
        raise ContractError(
            f"head_dim mismatch: q {q.shape[2]}, k {k.shape[2]}, shape.head_dim {shape.head_dim}"
        )
    if k.shape[:2] != v.shape[:2] or v.shape[2] != shape.head_dim:
        raise ContractError(f"k/v shape mismatch: {tuple(k.shape)} vs {tuple(v.shape)}")
    if k.shape[0] != q.shape[0]:
        raise ContractError(f"k has {k.shape[0]} heads, q has {q.shape[0]}")
    q, k, v = (t.contiguous() for t in _promote(q, k, v))
    out, lse, w = attend_dense_dev(q, k, v, float(shape.scale), keep_weights)
    if single:
        out, lse = out[0], lse[0]
        w = w[0] if w is not None else None
    return AttentionResult(back(out, np_q), back(lse, np_q), back(w, np_q) if w is not None else None)


def attend_dense_dev(q, k, v, scale, keep_weights):
    """Backend contract on device tensors: q [H,nq,d], k/v [H,nkv,d]."""
    H, nq, d = q.shape
    nkv = k.shape[1]
    dev = q.device
    out = torch.zeros((H, nq, d), dtype=q.dtype, device=dev)
    lse = torch.full((H, nq), -math.inf, dtype=torch.float64, device=dev)
    w = torch.zeros((H, nq, nkv), dtype=q.dtype, device=dev) if keep_weights else None
    if H * nq == 0:
        return out, lse, w
    ws = torch.empty(max(H * nq * max(nkv, 1), 1), dtype=torch.float64, device=dev)
    _lib.call("hgca_attend_dense", DTYPE_CODE[q.dtype], q.data_ptr(), k.data_ptr() if nkv else None,
              v.data_ptr() if nkv else None, H, nq, nkv, d, scale, int(keep_weights),
              out.data_ptr(), lse.data_ptr(), w.data_ptr() if (w is not None and nkv) else None,
              ws.data_ptr(), stream_handle(dev))
    return out, lse, w


def attend_indexed(q, k, v, idx, scale: float, keep_weights: bool = False) -> AttentionResult:
    """Single-head gathered attention (attention.py:127-150)."""
    (q, np_q), (k, _), (v, _) = _working(q, "q"), _working(k, "k"), _working(v, "v")
    if q.dim() != 2 or k.dim() != 2 or v.dim() != 2:
        raise ContractError("attend_indexed takes single-head 2-D arrays")
    if k.shape != v.shape or q.shape[1] != k.shape[1]:
        raise ContractError(
            f"incompatible shapes: q {tuple(q.shape)}, k {tuple(k.shape)}, v {tuple(v.shape)}"
        )
    if isinstance(idx, torch.Tensor):
        idx_t = idx.to(device=q.device, dtype=torch.int64).contiguous()
        idx_np = None
    else:
        idx_np = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        idx_t = None
    n = int(idx_np.size if idx_np is not None else idx_t.numel())
    if n:
        lo_hi = (idx_np.min(), idx_np.max()) if idx_np is not None else (int(idx_t.min()), int(idx_t.max()))
        if lo_hi[0] < 0 or lo_hi[1] >= k.shape[0]:
            raise ContractError("idx out of bounds")
    if idx_t is None:
        idx_t = torch.from_numpy(idx_np).to(q.device)
    q, k, v = (t.contiguous() for t in _promote(q, k, v))
    out, lse, w = attend_indexed_dev(q, k, v, idx_t, float(scale), keep_weights)
    return AttentionResult(back(out, np_q), back(lse, np_q), back(w, np_q) if w is not None else None)


def attend_indexed_dev(q, k, v, idx, scale, keep_weights):
    nq, d = q.shape
    n = idx.numel()
    M = k.shape[0]
    dev = q.device
    out = torch.zeros((nq, d), dtype=q.dtype, device=dev)
    lse = torch.full((nq,), -math.inf, dtype=torch.float64, device=dev)
    w = torch.zeros((nq, n), dtype=q.dtype, device=dev) if keep_weights else None
    if nq == 0:
        return out, lse, w
    ws = torch.empty(max(nq * max(n, 1), 1), dtype=torch.float64, device=dev)
    _lib.call("hgca_attend_indexed", DTYPE_CODE[q.dtype], q.data_ptr(),
              k.data_ptr() if M else None, v.data_ptr() if M else None,
              idx.data_ptr() if n else None, n, M, nq, d, scale, int(keep_weights),
              out.data_ptr(), lse.data_ptr(), w.data_ptr() if (w is not None and n) else None,
              ws.data_ptr(), stream_handle(dev))
    return out, lse, w


def merge_states(a: AttentionResult, b: AttentionResult) -> AttentionResult:
    """Exact LSE merge of two partials over disjoint key sets (attention.py:153-188)."""
    oa, np_a = as_device(a.output)
    ob, _ = as_device(b.output)
    la, _ = as_device(a.lse)
    lb, _ = as_device(b.lse)
    if tuple(oa.shape) != tuple(ob.shape):
        raise ContractError(f"output shape mismatch: {tuple(oa.shape)} vs {tuple(ob.shape)}")
    if tuple(la.shape) != tuple(lb.shape):
        raise ContractError(f"lse shape mismatch: {tuple(la.shape)} vs {tuple(lb.shape)}")
    dt = torch.float64 if torch.float64 in (oa.dtype, ob.dtype) else torch.float32
    if oa.dtype not in (torch.float32, torch.float64) or ob.dtype not in (torch.float32, torch.float64):
        dt = torch.float64
    oa = oa.to(dt).contiguous()
    ob = ob.to(dt).contiguous()
    la = la.to(torch.float64).contiguous()
    lb = lb.to(torch.float64).contiguous()
    d = oa.shape[-1] if oa.dim() else 1
    rows = la.numel()
    out = torch.empty_like(oa)
    lse = torch.empty_like(la)
    wa = wb = wout = None
    na = nb = 0
    if a.weights is not None and b.weights is not None:
        wa, _ = as_device(a.weights)
        wb, _ = as_device(b.weights)
        wa = wa.to(dt).contiguous()
        wb = wb.to(dt).contiguous()
        na, nb = wa.shape[-1], wb.shape[-1]
        wout = torch.empty(tuple(wa.shape[:-1]) + (na + nb,), dtype=dt, device=oa.device)
    if rows:
        _lib.call("hgca_merge_states", DTYPE_CODE[dt], oa.data_ptr(), la.data_ptr(), ob.data_ptr(),
                  lb.data_ptr(), rows, d, out.data_ptr(), lse.data_ptr(),
                  wa.data_ptr() if wa is not None else None,
                  wb.data_ptr() if wb is not None else None, na, nb,
                  wout.data_ptr() if wout is not None and (na + nb) else None,
                  stream_handle(oa.device))
    return AttentionResult(back(out, np_a), back(lse, np_a), back(wout, np_a) if wout is not None else None)


def logsumexp(scores) -> float:
    """attention.py:191-199. A host-side scalar utility in the reference (not on
    the engine path); kept on the host here too."""
    s = np.asarray(scores.detach().cpu() if isinstance(scores, torch.Tensor) else scores,
                   dtype=np.float64).ravel()
    if s.size == 0:
        return float("-inf")
    m = s.max()
    if not np.isfinite(m):
        return float(m)
    return float(m + np.log(np.exp(s - m).sum()))


__all__ += ["attend_dense_dev", "attend_indexed_dev", "device"]

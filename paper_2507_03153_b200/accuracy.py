"""Full-attention reference and the reference harness's accuracy metrics, on the GPU.

The reference checks the hybrid step against an fp64 softmax attention over the
whole history (oracle.py:27-55) and reports, per head (harness.py:135-160):

  * err   = |out_hybrid - out_full|                      (max / mean over dims)
  * eps   = 1 - (oracle weight mass on the attended set)  (the dropped mass)
  * bound = 2 * eps * max|V|  per dim; a head violates it when err - bound > slack

Here the full attention runs through libhgca_b200 (hgca_attend_gqa: fp64 dot
products in the reference's order, exact fp64 softmax, float32 weights) over
every written position of a layer, and the attended set is the step's window
plus its selected archive entries, read from the engine's selection masks.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .errors import ContractError

__all__ = ["full_attention", "attended_mask", "step_metrics"]


def full_attention(eng, layer_idx, q, n):
    """fp64 attention of q [B, Hq, 1, D] (storage dtype, on the device) over
    positions [0, n) of the layer -> (out [B*Hq, D] f32, lse [B*Hq] f64,
    weights [B*Hq, n] f64)."""
    ls = eng.layers[layer_idx]
    BHq = eng.B * eng.Hq
    if not 0 < n <= ls.nxt:
        raise ContractError(f"full_attention over [0, {n}) but only {ls.nxt} positions are written")
    q = q.to(device=eng.dev, dtype=eng.tdtype).contiguous()
    out = torch.empty((BHq, 1, eng.D), dtype=torch.float32, device=eng.dev)
    lse = torch.empty((BHq, 1), dtype=torch.float64, device=eng.dev)
    w = torch.empty((BHq, 1, n), dtype=torch.float32, device=eng.dev)
    ws = torch.empty(BHq * n, dtype=torch.float64, device=eng.dev)
    _lib.call("hgca_attend_gqa", eng.dcode, q.data_ptr(), ls.KV.data_ptr(), eng.B, eng.Hq, eng.Hkv, eng.T, 0, n, 1,
              eng.D, float(eng.shape.scale), out.data_ptr(), lse.data_ptr(), w.data_ptr(), n, ws.data_ptr(),
              eng._stream())
    # fp64 weights for the mass accounting: ws holds exp(s - m) per key (fp64)
    e = ws.view(BHq, n)
    return out[:, 0], lse[:, 0], e / e.sum(dim=1, keepdim=True)


def attended_mask(eng, layer_idx, n):
    """[B*Hq, n] bool: the positions the next decode step attends -- its
    selected archive entries (context + padding) and the window plus the new
    token (positions [lo, n))."""
    ls = eng.layers[layer_idx]
    words = ls.sel.shape[1]
    bits = torch.arange(32, device=eng.dev, dtype=torch.int64)
    sel = ((ls.sel.to(torch.int64)[:, :, None] >> bits) & 1).bool().reshape(ls.sel.shape[0], words * 32)
    mask = torch.zeros((ls.sel.shape[0], n), dtype=torch.bool, device=eng.dev)
    mask[:, : ls.lo] = sel[:, : ls.lo]
    mask[:, ls.lo: n] = True
    return mask


def step_metrics(eng, layer_idx, out_hybrid, q, mask, n, slack=1e-5):
    """harness.py:147-160 for one decode step: out_hybrid [B*Hq, D] is the
    step's output for queries q over positions [0, n), mask the attended set
    (attended_mask taken before the step)."""
    out_f, _, w = full_attention(eng, layer_idx, q, n)
    err = (out_hybrid.double() - out_f.double()).abs()                     # [BHq, D]
    retained = (w * mask.double()).sum(dim=1)
    eps = (1.0 - retained).clamp(min=0.0)
    ls = eng.layers[layer_idx]
    vabs = ls.rows()[:, :n, 1].double().abs().amax(dim=1)                 # [B*Hkv, D]
    G = eng.Hq // eng.Hkv
    b = torch.arange(eng.B * eng.Hq, device=eng.dev) // eng.Hq
    h = torch.arange(eng.B * eng.Hq, device=eng.dev) % eng.Hq
    vabs_q = vabs[b * eng.Hkv + h // G]                                     # [BHq, D]
    bound = 2.0 * eps[:, None] * vabs_q
    gap = (err - bound).amax(dim=1)
    return {
        "max_err": float(err.max()), "mean_err": float(err.mean()),
        "eps_max": float(eps.max()), "eps_mean": float(eps.mean()),
        "bound_violations": int((gap > slack).sum()), "heads": int(eps.numel()),
        "attended_frac": float(mask.double().mean()),
        "max_gap": float(gap.max()) if math.isfinite(float(gap.max())) else None,
    }

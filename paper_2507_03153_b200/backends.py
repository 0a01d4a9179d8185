"""The `cuda` backend for the reference's kernel plugin slot.

tierkv selects its attention kernels through a module-level namespace
(backends.py:8-20, 65-100): `name`, `attend_dense(q, k, v, scale,
keep_weights)` and `attend_indexed(q, k, v, idx, scale, keep_weights)` on
C-contiguous numpy arrays, returning (out in the input dtype, lse float64,
weights or None). CUDA below implements exactly that contract on the B200;
install() registers it in a tierkv.backends module and makes it active, after
which tierkv's own attend / attend_indexed / HybridEngine run on the GPU.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from .attention import attend_dense_dev, attend_indexed_dev
from ._dev import device


def _cuda_attend_dense(q, k, v, scale, keep_weights):
    dev = device()
    dt = q.dtype
    tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (q, k, v))
    out, lse, w = attend_dense_dev(tq, tk, tv, float(scale), bool(keep_weights))
    res = (out.cpu().numpy().astype(dt, copy=False), lse.cpu().numpy(),
           w.cpu().numpy().astype(dt, copy=False) if w is not None else None)
    return res


def _cuda_attend_indexed(q, k, v, idx, scale, keep_weights):
    dev = device()
    dt = q.dtype
    tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (q, k, v))
    ti = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int64)).to(dev)
    out, lse, w = attend_indexed_dev(tq, tk, tv, ti, float(scale), bool(keep_weights))
    return (out.cpu().numpy().astype(dt, copy=False), lse.cpu().numpy(),
            w.cpu().numpy().astype(dt, copy=False) if w is not None else None)


CUDA = SimpleNamespace(name="cuda", attend_dense=_cuda_attend_dense, attend_indexed=_cuda_attend_indexed)


def install(backends_module=None, activate: bool = True):
    """Register CUDA in tierkv.backends._BACKENDS and optionally activate it.

    Mirrors what a reference maintainer would add next to `_BACKENDS`
    (backends.py:71-77); `active` is read at call time by attention.py:118/147.
    """
    if backends_module is None:
        import tierkv.backends as backends_module  # noqa: PLC0415  (reference package)
    backends_module._BACKENDS["cuda"] = CUDA
    if activate:
        backends_module.active = CUDA
    return CUDA

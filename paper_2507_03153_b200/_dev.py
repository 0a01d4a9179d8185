"""Device plumbing: host<->HBM movement and stream handles (torch is used for
device memory and streams only; all arithmetic runs in libhgca_b200.so)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

DTYPE_CODE = {torch.float32: _lib.DTYPE_F32, torch.float64: _lib.DTYPE_F64, torch.bfloat16: _lib.DTYPE_BF16}


def device():
    """The CUDA device used by the product path; raises without a GPU."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2507_03153_b200 requires a CUDA device (no CPU fallback)")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def as_device(x):
    """(tensor on the CUDA device, came_from_numpy)."""
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            return x.to(device()), False
        return x, False
    a = np.asarray(x)
    if a.dtype == object:
        a = a.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device()), True


def back(t, to_numpy):
    if t is None or not to_numpy:
        return t
    return t.detach().cpu().numpy()


def stream_handle(dev=None):
    return torch.cuda.current_stream(dev).cuda_stream

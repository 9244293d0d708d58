"""Device plumbing: torch owns device memory and streams; kernels are ours."""

from __future__ import annotations

import numpy as np


def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_2505_03728_b200 computes on a CUDA device (sm_100a) only; no GPU is visible "
            "and there is no CPU fallback")
    return t


def stream_handle() -> int:
    t = require_cuda()
    return int(t.cuda.current_stream().cuda_stream)


def to_dev(x, dtype=None):
    """Contiguous device tensor (float64 by default) from numpy / lists / tensors."""
    t = require_cuda()
    dtype = dtype or t.float64
    if isinstance(x, t.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    return t.as_tensor(np.ascontiguousarray(x), dtype=dtype).to("cuda").contiguous()


def empty(shape, dtype=None):
    t = require_cuda()
    return t.empty(shape, dtype=dtype or t.float64, device="cuda")


def ptr(x) -> int | None:
    return None if x is None else int(x.data_ptr())

"""Device plumbing for the API layer: numpy/torch inputs -> CUDA tensors.

PyTorch only holds device memory and streams here; every computation is a
libct kernel.  numpy inputs are copied in and results copied back (parity
mode, how the reference's tests call the API); torch CUDA inputs stay on the
device.
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import CT_F64, CT_U8, CT_U16

_NP_TO_TORCH = {
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.uint16): torch.uint16,
    np.dtype(np.float64): torch.float64,
}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1407_2089_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_device(values, allow=(torch.uint8, torch.uint16, torch.float64)) -> torch.Tensor:
    """Contiguous CUDA tensor; dtypes outside `allow` become float64 (the
    reference casts with ``astype(np.float64)``, ref denoise.py:84)."""
    dev = require_cuda()
    if isinstance(values, torch.Tensor):
        t = values
        if t.dtype == torch.bool:
            t = t.to(torch.uint8)
        if t.dtype not in allow:
            t = t.to(device=dev).to(torch.float64)
        return t.to(device=dev).contiguous()
    a = np.asarray(values)
    if a.dtype == np.bool_:
        a = a.astype(np.uint8)
    tdt = _NP_TO_TORCH.get(a.dtype)
    if tdt is None or tdt not in allow:
        a = a.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def ct_code(t: torch.Tensor) -> int:
    return {torch.uint8: CT_U8, torch.uint16: CT_U16, torch.float64: CT_F64}[t.dtype]


def empty(shape, dtype, device=None) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device or require_cuda())


def zeros(shape, dtype, device=None) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device or require_cuda())


def like_input(result: torch.Tensor, template):
    """numpy in -> numpy out; torch in -> torch out."""
    if isinstance(template, torch.Tensor):
        return result
    if result.dtype == torch.uint16:
        return result.cpu().view(torch.int16).numpy().view(np.uint16)
    return result.cpu().numpy()

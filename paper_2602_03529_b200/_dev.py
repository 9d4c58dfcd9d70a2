"""Device plumbing for the numpy-facing API: torch owns device memory and the
current CUDA stream; the kernels run through the C ABI (``_lib``)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("semstream_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() > 0 else None


def h2d(a: np.ndarray, dtype=None) -> torch.Tensor:
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    if not arr.flags.writeable:          # torch.from_numpy needs a writable buffer
        arr = arr.copy()
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(tuple(shape), dtype=dtype, device=device())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(tuple(shape), dtype=dtype, device=device())


def d2h(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()

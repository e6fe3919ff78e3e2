"""Host<->device plumbing shared by the API modules (torch owns memory and streams)."""

from __future__ import annotations

import contextlib
import warnings

import numpy as np
import torch

from . import _native


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise _native.NativeUnavailable("a CUDA device is required (the product path has no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def as_cuda(x, dtype=None) -> torch.Tensor:
    """numpy / torch -> contiguous-innermost CUDA tensor (copy only when needed)."""
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(device(), non_blocking=False)
    else:
        a = np.ascontiguousarray(x)
        with warnings.catch_warnings():  # read-only (frozen) arrays are only read here
            warnings.simplefilter("ignore", UserWarning)
            t = torch.from_numpy(a).to(device())
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t


def is_numpy(x) -> bool:
    return isinstance(x, np.ndarray)


def to_like(t: torch.Tensor, like):
    """Return numpy if the caller passed numpy, else the tensor."""
    if is_numpy(like):
        return t.cpu().numpy()
    return t


def code_of(dtype: torch.dtype, allow_f64: bool = False) -> int:
    if dtype == torch.float64 and allow_f64:
        return _native.F64
    if dtype == torch.float32:
        return _native.F32
    if dtype == torch.bfloat16:
        return _native.BF16
    if dtype == torch.float16:
        return _native.F16
    raise TypeError(f"unsupported dtype {dtype} (float32, bfloat16 or float16)")


def stream() -> int:
    """The current stream of the current device (callers enter ``on(t)`` first)."""
    return torch.cuda.current_stream().cuda_stream


def on(t):
    """Make ``t``'s device current for the native calls in the block (launches go to that
    device's current stream, and the C side's cudaGetDevice queries the same device)."""
    if isinstance(t, torch.Tensor) and t.is_cuda:
        return torch.cuda.device(t.device)
    return contextlib.nullcontext()


def same_device(*ts) -> None:
    """ShapeError unless every tensor lives on one device."""
    devs = {t.device for t in ts if isinstance(t, torch.Tensor)}
    if len(devs) > 1:
        from .errors import ShapeError

        raise ShapeError(f"tensors live on different devices: {sorted(map(str, devs))}")

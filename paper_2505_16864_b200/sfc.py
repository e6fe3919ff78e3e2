"""Space-filling-curve orderings on the GPU (reference: tokencarve sfc.py).

``build_curve`` runs the K1 kernel (``tcb_curve_build``): every cell computes its
own position on the slab-paired generalized-Hilbert curve by descending the
gilbert split tree, so the permutation is built in one launch instead of the
reference's recursive emission (sfc.py:98-210).  ``apply_permutation`` /
``invert_permutation`` run the K2 gather (``tcb_gather_rows``), 16-byte
vectorised, any row payload (sfc.py:213-237).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _native
from .errors import ShapeError, SizeError

__all__ = ["GridDims", "Permutation", "build_curve", "apply_permutation", "invert_permutation",
           "padded_token_count"]

_MAX_CELLS = 2**31 - 1  # int32 device indices (reference: 2**62, sfc.py:38)


@dataclass(frozen=True)
class GridDims:
    """(t, h, w) latent grid, validated like sfc.py:41-67."""

    t: int
    h: int
    w: int

    def __post_init__(self):
        for name in ("t", "h", "w"):
            v = getattr(self, name)
            if not isinstance(v, (int, np.integer)) or isinstance(v, bool) or v < 1:
                raise ShapeError(f"grid axis {name} must be a positive integer, got {v!r}")

    @property
    def n_cells(self) -> int:
        return int(self.t) * int(self.h) * int(self.w)

    def as_tuple(self) -> tuple[int, int, int]:
        return (int(self.t), int(self.h), int(self.w))

    @classmethod
    def from_string(cls, text: str) -> "GridDims":
        parts = text.replace("x", ",").split(",")
        if len(parts) != 3:
            raise ShapeError(f"expected 't,h,w', got {text!r}")
        return cls(*(int(p) for p in parts))


class Permutation:
    """Curve <-> row-major bijection (sfc.py:70-95).

    ``forward[i]`` is the row-major cell at curve position i; ``inverse`` its inverse.
    As in the reference both are read-only int64 numpy arrays (sfc.py:91-92; copied
    from the device once, on first access).  The kernels use the device copies
    ``forward_dev`` / ``inverse_dev`` (int32, resident in HBM).  Immutable like the
    reference's frozen dataclass.
    """

    __slots__ = ("dims", "forward_dev", "inverse_dev", "_np")

    def __init__(self, dims: GridDims, forward, inverse):
        n = dims.n_cells
        if tuple(forward.shape) != (n,) or tuple(inverse.shape) != (n,):
            raise ShapeError(f"permutation arrays must have length {n}, got "
                             f"{tuple(forward.shape)} / {tuple(inverse.shape)}")
        fwd = _dev.as_cuda(forward, torch.int32)
        inv = _dev.as_cuda(inverse, torch.int32)
        host = {}
        if not isinstance(forward, torch.Tensor) or not isinstance(inverse, torch.Tensor):
            # a caller-built permutation is checked like sfc.py:88-89
            f64 = np.asarray(forward.cpu() if isinstance(forward, torch.Tensor) else forward,
                             dtype=np.int64)
            i64 = np.asarray(inverse.cpu() if isinstance(inverse, torch.Tensor) else inverse,
                             dtype=np.int64)
            if not np.array_equal(f64[i64], np.arange(n)):
                raise ShapeError("inverse is not the inverse of forward")
        for name, val in (("dims", dims), ("forward_dev", fwd), ("inverse_dev", inv), ("_np", host)):
            object.__setattr__(self, name, val)

    def __setattr__(self, name, value):
        raise AttributeError(f"Permutation is immutable (cannot set {name!r})")

    def __len__(self) -> int:
        return int(self.forward_dev.shape[0])

    def __repr__(self) -> str:
        return f"Permutation(dims={self.dims!r}, n={len(self)})"

    def _host(self, key: str, dev: torch.Tensor) -> np.ndarray:
        a = self._np.get(key)
        if a is None:
            a = dev.cpu().numpy().astype(np.int64)
            a.setflags(write=False)
            self._np[key] = a
        return a

    @property
    def forward(self) -> np.ndarray:
        return self._host("f", self.forward_dev)

    @property
    def inverse(self) -> np.ndarray:
        return self._host("i", self.inverse_dev)

    # round-1 names, kept for callers of this package
    forward_np = forward
    inverse_np = inverse


def build_curve(dims: GridDims) -> Permutation:
    """Curve permutation for ``dims`` (sfc.py:198-210), one K1 launch."""
    n = dims.n_cells
    if n > _MAX_CELLS:
        raise SizeError(f"{n} cells exceed the supported index range")
    dev = _dev.device()
    fwd = torch.empty(n, dtype=torch.int32, device=dev)
    inv = torch.empty(n, dtype=torch.int32, device=dev)
    _native.call("tcb_curve_build", dims.t, dims.h, dims.w, fwd.data_ptr(), inv.data_ptr(),
                 _dev.stream())
    perm = Permutation.__new__(Permutation)
    for name, val in (("dims", dims), ("forward_dev", fwd), ("inverse_dev", inv), ("_np", {})):
        object.__setattr__(perm, name, val)
    return perm


def gather_rows(x: torch.Tensor, index: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[i] = x[index[i]] along axis 0 for any contiguous payload (K2)."""
    if not x.is_contiguous():
        x = x.contiguous()
    rows = index.shape[0]
    if out is None:
        out = torch.empty((rows, *x.shape[1:]), dtype=x.dtype, device=x.device)
    row_bytes = x[0].numel() * x.element_size() if x.shape[0] else 0
    _native.call("tcb_gather_rows", x.data_ptr(), out.data_ptr(), index.data_ptr(), rows, row_bytes,
                 x.shape[0], _dev.stream())
    return out


def _permute(tokens, index: torch.Tensor):
    n = index.shape[0]
    if isinstance(tokens, (np.ndarray, torch.Tensor)):
        if tokens.shape[0] != n:
            raise ShapeError(f"sequence length {tokens.shape[0]} != permutation length {n}")
        t = _dev.as_cuda(tokens)
        return _dev.to_like(gather_rows(t, index), tokens)
    seq = list(tokens)
    if len(seq) != n:
        raise ShapeError(f"sequence length {len(seq)} != permutation length {n}")
    return [seq[i] for i in index.cpu().tolist()]


def apply_permutation(tokens, perm: Permutation):
    """Curve order: ``out[i] = tokens[perm.forward[i]]`` (sfc.py:226-232)."""
    return _permute(tokens, perm.forward_dev)


def invert_permutation(tokens, perm: Permutation):
    """Row-major order: ``out[i] = tokens[perm.inverse[i]]`` (sfc.py:235-237)."""
    return _permute(tokens, perm.inverse_dev)


def padded_token_count(n_tokens: int, m: int) -> tuple[int, int]:
    """Smallest multiple of m >= n_tokens, and the pad (sfc.py:240-251)."""
    if m < 1:
        raise ShapeError(f"block size must be >= 1, got {m}")
    if n_tokens < 1:
        raise ShapeError(f"token count must be >= 1, got {n_tokens}")
    padded = -(-n_tokens // m) * m
    return padded, padded - n_tokens

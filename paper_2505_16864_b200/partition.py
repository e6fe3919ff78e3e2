"""Block layout of the curve-ordered token stream and the static block masks
(reference: tokencarve partition.py).

Layout ``[vision | vision pad | cond | cond pad]`` in curve positions
(partition.py:3-13).  The kernels never read a validity tensor: validity is a
prefix of every block and is derived in-kernel from ``(m, M_v, n_valid,
n_cond)``.  The 26-neighbour adjacency is built on the device by K6 into a
packed bitset whose row stride (``words``) equals the selection mask's, so the
union in the selection kernel is a word-wise OR.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _dev, _native
from .errors import ShapeError
from .sfc import GridDims, Permutation, padded_token_count

__all__ = ["BlockLayout", "StaticMasks", "build_layout", "adjacency_mask", "condition_mask",
           "mask_words"]


def mask_words(M_total: int) -> int:
    """uint32 words per packed mask row."""
    return max(1, -(-M_total // 32))


@dataclass(frozen=True)
class BlockLayout:
    """Block bookkeeping for one (dims, m, n_cond) (partition.py:38-88)."""

    m: int
    n_valid: int
    n_cond: int
    M_v: int
    M_c: int

    @property
    def M_total(self) -> int:
        return self.M_v + self.M_c

    @property
    def padded_vision(self) -> int:
        return self.M_v * self.m

    @property
    def padded_total(self) -> int:
        return self.M_total * self.m

    @property
    def cond_start(self) -> int:
        return self.padded_vision

    @property
    def valid_len(self) -> int:
        return self.n_valid + self.n_cond

    @cached_property
    def cell_to_block(self) -> np.ndarray:
        return np.arange(self.padded_total, dtype=np.int64) // self.m

    @cached_property
    def token_valid_mask(self) -> np.ndarray:
        mask = np.zeros(self.padded_total, dtype=bool)
        mask[: self.n_valid] = True
        mask[self.cond_start: self.cond_start + self.n_cond] = True
        mask.setflags(write=False)
        return mask

    @cached_property
    def block_valid_counts(self) -> np.ndarray:
        idx = np.arange(self.M_total, dtype=np.int64)
        vis = np.clip(self.n_valid - idx * self.m, 0, self.m)
        cond = np.clip(self.n_cond - (idx - self.M_v) * self.m, 0, self.m)
        counts = np.where(idx < self.M_v, vis, cond)
        counts.setflags(write=False)
        return counts


def build_layout(dims: GridDims, m: int, n_cond_tokens: int = 0) -> BlockLayout:
    """partition.py:91-104."""
    if m < 1:
        raise ShapeError(f"block size must be >= 1, got {m}")
    if n_cond_tokens < 0:
        raise ShapeError(f"condition token count must be >= 0, got {n_cond_tokens}")
    n_valid = dims.n_cells
    padded_v, _ = padded_token_count(n_valid, m)
    m_c = padded_token_count(n_cond_tokens, m)[0] // m if n_cond_tokens else 0
    return BlockLayout(m=m, n_valid=n_valid, n_cond=n_cond_tokens, M_v=padded_v // m, M_c=m_c)


def adjacency_bits(layout: BlockLayout, dims: GridDims, perm: Permutation) -> torch.Tensor:
    """Packed (M_v, words) uint32 adjacency on the device, one K6 launch."""
    if perm.dims != dims:
        raise ShapeError("permutation was built for different dims")
    if layout.n_valid != dims.n_cells:
        raise ShapeError("layout was built for different dims")
    words = mask_words(layout.M_total)
    inv = perm.inverse_dev
    with _dev.on(inv):
        out = torch.empty((layout.M_v, words), dtype=torch.int32, device=inv.device)
        _native.call("tcb_adjacency_build", inv.data_ptr(), dims.t, dims.h, dims.w, layout.m,
                     layout.M_v, words, out.data_ptr(), _dev.stream())
    return out


def unpack_rows(bits: torch.Tensor, n_cols: int) -> torch.Tensor:
    """Packed uint32 rows -> dense bool (..., n_cols) on the device."""
    lead = bits.shape[:-1]
    rows = int(np.prod(lead)) if len(lead) else 1
    with _dev.on(bits):
        out = torch.empty((*lead, n_cols), dtype=torch.uint8, device=bits.device)
        _native.call("tcb_mask_unpack", bits.data_ptr(), rows, n_cols, bits.shape[-1],
                     out.data_ptr(), _dev.stream())
    return out.view(torch.bool)


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


def adjacency_mask(layout: BlockLayout, dims: GridDims, perm: Permutation) -> np.ndarray:
    """Dense bool (M_v, M_v) adjacency (partition.py:107-136): built on the device by K6,
    returned as numpy like the reference."""
    dense = unpack_rows(adjacency_bits(layout, dims, perm), layout.M_total)[:, : layout.M_v]
    return dense.cpu().numpy()


def condition_mask(layout: BlockLayout) -> np.ndarray:
    """``i >= M_v or j >= M_v`` (partition.py:139-143); a host array like the reference
    (the device path never materialises it: the select kernel forces the columns)."""
    is_cond = np.arange(layout.M_total) >= layout.M_v
    return is_cond[:, None] | is_cond[None, :]


class StaticMasks:
    """Per-stage masks (partition.py:146-159).

    ``adja_bits`` is the packed (M_v, words) device bitset the selection kernel ORs in;
    ``cond`` / ``adja`` are the reference's read-only dense bool numpy arrays
    (partition.py:154-155), materialised from the device on first access;
    ``cond_dev`` / ``adja_dev`` are the dense device views.
    """

    __slots__ = ("_cond", "_adja", "adja_bits", "_cache")

    def __init__(self, cond=None, adja=None, adja_bits: torch.Tensor | None = None):
        if adja is None and adja_bits is None:
            raise ShapeError("StaticMasks needs adja (dense) or adja_bits (packed)")
        object.__setattr__(self, "_cond", cond)
        object.__setattr__(self, "_adja", adja)
        object.__setattr__(self, "adja_bits", adja_bits)
        object.__setattr__(self, "_cache", {})
        for a in (cond, adja):
            if isinstance(a, np.ndarray):
                a.setflags(write=False)

    def __setattr__(self, name, value):
        raise AttributeError(f"StaticMasks is immutable (cannot set {name!r})")

    def __repr__(self) -> str:
        return f"StaticMasks(M_v={self.adja_dev.shape[0]})"

    @classmethod
    def build(cls, layout: BlockLayout, dims: GridDims, perm: Permutation) -> "StaticMasks":
        bits = adjacency_bits(layout, dims, perm)
        sm = cls(cond=None, adja=None, adja_bits=bits)
        sm._cache["M_total"] = layout.M_total
        sm._cache["M_v"] = layout.M_v
        return sm

    def _get(self, key, make):
        v = self._cache.get(key)
        if v is None:
            v = make()
            self._cache[key] = v
        return v

    @property
    def adja_dev(self) -> torch.Tensor:
        if isinstance(self._adja, torch.Tensor):
            return self._adja
        if self._adja is not None:
            return self._get("adja_dev", lambda: _dev.as_cuda(self._adja).to(torch.bool))
        M_v, M_total = self._cache["M_v"], self._cache["M_total"]
        return self._get("adja_dev", lambda: unpack_rows(self.adja_bits, M_total)[:, :M_v])

    @property
    def adja(self) -> np.ndarray:
        if isinstance(self._adja, np.ndarray):
            return self._adja
        return self._get("adja_np", lambda: _frozen(self.adja_dev.cpu().numpy()))

    @property
    def cond(self) -> np.ndarray:
        if isinstance(self._cond, np.ndarray):
            return self._cond
        if isinstance(self._cond, torch.Tensor):
            return self._get("cond_np", lambda: _frozen(self._cond.cpu().numpy()))
        M_v, M_total = self._cache["M_v"], self._cache["M_total"]
        return self._get("cond_np", lambda: _frozen(condition_mask(
            BlockLayout(m=1, n_valid=M_v, n_cond=M_total - M_v, M_v=M_v, M_c=M_total - M_v))))

    @property
    def cond_dev(self) -> torch.Tensor:
        if isinstance(self._cond, torch.Tensor):
            return self._cond
        return self._get("cond_dev", lambda: _dev.as_cuda(self.cond))

    def packed(self, layout: BlockLayout) -> torch.Tensor:
        """The (M_v, words) packed adjacency the selection kernel consumes."""
        if self.adja_bits is not None:
            return self.adja_bits

        def make():
            dense = torch.zeros((layout.M_v, layout.M_total), dtype=torch.uint8, device=_dev.device())
            dense[:, : layout.M_v] = self.adja_dev.to(torch.uint8)
            return pack_rows(dense, layout.M_total)[0]
        return self._get(("packed", layout.M_total), make)


def pack_rows(dense: torch.Tensor, n_cols: int):
    """Dense bool/uint8 (..., n_cols) -> (packed uint32 rows, row popcounts kv_cnt)."""
    d8 = dense.contiguous().view(torch.uint8) if dense.dtype == torch.bool else dense.contiguous()
    lead = d8.shape[:-1]
    rows = int(np.prod(lead)) if len(lead) else 1
    words = mask_words(n_cols)
    with _dev.on(d8):
        bits = torch.empty((*lead, words), dtype=torch.int32, device=d8.device)
        kv_cnt = torch.empty(lead, dtype=torch.int32, device=d8.device)
        _native.call("tcb_mask_pack", d8.data_ptr(), rows, n_cols, words, bits.data_ptr(),
                     kv_cnt.data_ptr(), _dev.stream())
    return bits, kv_cnt

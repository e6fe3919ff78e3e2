"""Dynamic block selection on the GPU (reference: tokencarve masks.py).

``build_block_mask`` runs K3 ``tcb_block_pool`` (Q and K in one pass, float64
accumulation -> pooled means bit-exact with masks.py:112-116) and then either
* (R wanted -- the reference's return value) K4a ``tcb_block_scores`` (float64 pooled
  scores / sqrt(d), masks.py:130-131) and ``tcb_block_select_scores`` (row softmax with
  numpy's pairwise sums, masks.py:132-134, radix-select of the top n_keep under the stable
  descending order, the exact sequential prefix cutoff, and the union with the condition
  columns and the packed adjacency, masks.py:137-175), R left in place; or
* (``need_relevance=False``: the layer path) ``tcb_block_mask``: the same scores into a
  bounded scratch (never an R tensor beyond 256 MB) and the same selection; at p == 0 it
  selects on the scores themselves (the softmax is monotone) and re-runs near-tie rows
  through the exact softmax program.
The mask is packed (H, M_v, words) uint32 plus row counts; the attention kernel walks the
set bits of a row in ascending order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _native
from .errors import ContractError, ShapeError
from .partition import BlockLayout, StaticMasks, mask_words, pack_rows, unpack_rows

__all__ = ["PooledBlocks", "SelectionParams", "BlockMask", "block_pool", "relevance",
           "importance_mask", "union_mask", "build_block_mask", "mask_stats"]


@dataclass(frozen=True)
class PooledBlocks:
    """Per-head block means (H, blocks, d) float64 (masks.py:31-50).  ``values`` is a
    device tensor, or numpy when the caller pooled numpy input (as the reference)."""

    values: object
    valid_counts: np.ndarray

    def __post_init__(self):
        if self.values.ndim != 3:
            raise ShapeError(f"pooled values must be rank 3, got shape {tuple(self.values.shape)}")
        if tuple(self.valid_counts.shape) != (self.values.shape[1],):
            raise ShapeError("valid_counts length must equal the block count")

    @property
    def n_heads(self) -> int:
        return int(self.values.shape[0])

    @property
    def n_blocks(self) -> int:
        return int(self.values.shape[1])


@dataclass(frozen=True)
class SelectionParams:
    """Top-k rate and cutoff (masks.py:53-75)."""

    k: float = 0.3
    p: float = 0.3
    per_stage: tuple = (0.3, 0.2)

    def __post_init__(self):
        rates = (self.k, *self.per_stage)
        if any(not (0.0 < r <= 1.0) for r in rates):
            raise ContractError(f"selection rates must be in (0, 1], got {rates}")
        if not (0.0 <= self.p < 1.0):
            raise ContractError(f"cutoff probability must be in [0, 1), got {self.p}")

    def for_stage(self, stage: int) -> "SelectionParams":
        k = self.per_stage[min(stage, len(self.per_stage) - 1)]
        return SelectionParams(k=k, p=self.p, per_stage=self.per_stage)

    def n_floor(self, M_v: int) -> int:
        """Top-k quota max(1, ceil(k * M_v)) in float64 on the host (masks.py:154)."""
        return max(1, math.ceil(self.k * M_v))


class BlockMask:
    """Selection mask (H, M_v, M_total) (masks.py:78-95).

    Device form: packed ``words`` (H, M_v, ceil(M_total/32)) uint32 -- column j of a row is
    bit j % 32 of word j // 32 -- and the row counts ``kv_cnt`` (H, M_v).  The carve kernels
    walk a row's set bits in ascending order (the reference's flatnonzero, attention.py:179),
    so no index list is stored; ``kv_idx`` materialises the padded ascending lists on demand
    for inspection.  ``BlockMask(bits)``
    accepts a dense bool array/tensor like the reference and packs it on the device.
    ``.bits`` is the dense bool mask: a read-only numpy array when the mask came from
    numpy (a numpy ``bits`` argument, or ``build_block_mask`` on numpy Q/K), as the
    reference returns (masks.py:87); otherwise the device tensor (``bits_dev``).
    """

    def __init__(self, bits=None, *, words=None, kv_cnt=None, M_total=None,
                 nonempty: bool = False, host: bool | None = None):
        self._np = None
        if bits is not None:
            if bits.ndim != 3 or (bits.dtype not in (np.bool_, torch.bool)):
                raise ShapeError(f"mask bits must be a rank-3 boolean array, got {tuple(bits.shape)}")
            if isinstance(bits, np.ndarray):
                bits.setflags(write=False)  # the reference freezes the caller's array
                self._np = bits
            dense = _dev.as_cuda(bits)
            M_total = int(dense.shape[-1])
            words, kv_cnt = pack_rows(dense, M_total)
            self._dense = dense
            nonempty = False
            if host is None:
                host = isinstance(bits, np.ndarray)
        else:
            if words is None or kv_cnt is None or M_total is None:
                raise ShapeError("BlockMask needs bits= or the packed (words, kv_cnt)")
            self._dense = None
        self.words = words
        self.kv_cnt = kv_cnt
        self.M_total = int(M_total)
        self._nonempty = nonempty
        self.host = bool(host)

    @property
    def shape(self) -> tuple:
        return (*self.kv_cnt.shape, self.M_total)

    @property
    def bits_dev(self) -> torch.Tensor:
        """Dense bool (H, M_v, M_total) on the device (unpacked lazily)."""
        if self._dense is None:
            self._dense = unpack_rows(self.words, self.M_total)
        return self._dense

    @property
    def bits(self):
        if not self.host:
            return self.bits_dev
        if self._np is None:
            a = self.bits_dev.cpu().numpy()
            a.setflags(write=False)
            self._np = a
        return self._np

    @property
    def kv_idx(self) -> torch.Tensor:
        """(H, M_v, M_total) int32: row r's ascending kv blocks in its first kv_cnt[r] entries
        (the rest -1) -- derived from the bits on the device; the kernels never read it."""
        dense = self.bits_dev
        cols = torch.arange(self.M_total, dtype=torch.int32, device=dense.device)
        key = torch.where(dense, cols, torch.full_like(cols, self.M_total))
        srt = torch.sort(key, dim=-1).values
        return torch.where(srt < self.M_total, srt, torch.full_like(srt, -1))

    @property
    def n_heads(self) -> int:
        return int(self.kv_cnt.shape[0])

    @property
    def selected_fraction(self) -> float:
        total = int(np.prod(self.shape))
        return float(self.kv_cnt.sum().item()) / total if total else 0.0

    def check_nonempty(self) -> None:
        """ContractError on an empty row (attention.py:228-231); free for masks
        built by build_block_mask (the adjacency diagonal keeps rows non-empty)."""
        if self._nonempty or self.kv_cnt.numel() == 0:
            return
        mn = int(self.kv_cnt.min().item())
        if mn == 0:
            h, r = np.argwhere(self.kv_cnt.cpu().numpy() == 0)[0]
            raise ContractError(f"empty mask row for head {h}, query block {r}")
        self._nonempty = True


def _pool_one_or_two(x0: torch.Tensor, x1: torch.Tensor | None, layout: BlockLayout):
    for x in (x0,) if x1 is None else (x0, x1):
        if x.ndim != 3:
            raise ShapeError(f"expected (heads, tokens, d_k), got shape {tuple(x.shape)}")
        if x.shape[1] != layout.padded_total:
            raise ShapeError(f"token axis {x.shape[1]} != padded token count {layout.padded_total}")
    if x1 is not None and (x1.shape != x0.shape or x1.dtype != x0.dtype
                           or x1.stride() != x0.stride()):
        raise ShapeError("Q and K must share shape, dtype and strides")
    H, _, d = x0.shape
    if x0.stride(2) != 1:
        raise ShapeError("innermost (d_k) axis must be contiguous")
    if x1 is not None:
        _dev.same_device(x0, x1)
    with _dev.on(x0):
        outs = [torch.empty((H, layout.M_total, d), dtype=torch.float64, device=x0.device)
                for _ in range(1 if x1 is None else 2)]
        _native.call("tcb_block_pool", x0.data_ptr(), _native.ptr(x1),
                     _dev.code_of(x0.dtype, allow_f64=True), x0.stride(0), x0.stride(1), H, d,
                     layout.m, layout.M_v, layout.M_total, layout.n_valid, layout.n_cond,
                     outs[0].data_ptr(), outs[1].data_ptr() if x1 is not None else None,
                     _dev.stream())
    counts = layout.block_valid_counts.copy()
    return [PooledBlocks(values=o, valid_counts=counts) for o in outs]


def _poolable(x) -> torch.Tensor:
    """Device view of a pool input: 16/32/64-bit floats are read as they are; anything else
    (integer arrays) is promoted to float64 first, which is exact below 2^53."""
    t = _dev.as_cuda(x)
    if t.dtype not in (torch.float32, torch.bfloat16, torch.float16, torch.float64):
        t = t.to(torch.float64)
    return t


def block_pool(x, layout: BlockLayout) -> PooledBlocks:
    """Mean over valid tokens per block, float64 (masks.py:98-116).  numpy input (any float
    width, float64 included) gives numpy values, like the reference."""
    if x.ndim != 3:
        raise ShapeError(f"expected (heads, tokens, d_k), got shape {tuple(x.shape)}")
    pooled = _pool_one_or_two(_poolable(x), None, layout)[0]
    if _dev.is_numpy(x):
        return PooledBlocks(values=pooled.values.cpu().numpy(), valid_counts=pooled.valid_counts)
    return pooled


def relevance(pooled_q: PooledBlocks, pooled_k: PooledBlocks, d_k: int) -> torch.Tensor:
    """Row softmax of pooled scores / sqrt(d_k), float64 (masks.py:119-134)."""
    if pooled_q.n_heads != pooled_k.n_heads:
        raise ShapeError("pooled Q and K disagree on head count")
    if pooled_q.values.shape[2] != d_k or pooled_k.values.shape[2] != d_k:
        raise ShapeError("pooled Q/K feature size must equal d_k")
    pq = _dev.as_cuda(pooled_q.values, torch.float64).contiguous()
    pk = _dev.as_cuda(pooled_k.values, torch.float64).contiguous()
    _dev.same_device(pq, pk)
    H, rows, _ = pq.shape
    with _dev.on(pq):
        R = torch.empty((H, rows, pk.shape[1]), dtype=torch.float64, device=pq.device)
        _native.call("tcb_block_relevance", pq.data_ptr(), rows, pk.data_ptr(), H, rows,
                     pk.shape[1], d_k, R.data_ptr(), _dev.stream())
    return _dev.to_like(R, pooled_q.values)


def _select(R: torch.Tensor, params: SelectionParams, M_v: int, adja_bits, with_union: bool):
    H, rows, n_cols = R.shape
    words = mask_words(n_cols)
    dev = R.device
    with _dev.on(R):
        bits = torch.empty((H, rows, words), dtype=torch.int32, device=dev)
        kv_cnt = torch.empty((H, rows), dtype=torch.int32, device=dev)
        _native.call("tcb_block_select", R.data_ptr(), H, rows, n_cols, _native.ptr(adja_bits),
                     words, params.n_floor(M_v), float(params.p), 1 if with_union else 0,
                     bits.data_ptr(), kv_cnt.data_ptr(), _dev.stream())
    return bits, kv_cnt


def importance_mask(R, params: SelectionParams, M_v: int):
    """Cutoff + quota selection per row (masks.py:137-159); dense bool result."""
    if R.ndim != 3:
        raise ShapeError(f"relevance must be rank 3, got shape {tuple(R.shape)}")
    Rd = _dev.as_cuda(R, torch.float64).contiguous()
    bits, _ = _select(Rd, params, M_v, None, with_union=False)
    return _dev.to_like(unpack_rows(bits, Rd.shape[-1]), R)


def union_mask(b_top, cond, adja, layout: BlockLayout) -> BlockMask:
    """``b_top | cond[:M_v] | adja`` (masks.py:162-175)."""
    shape = (b_top.shape[0], layout.M_v, layout.M_total)
    if tuple(b_top.shape) != shape:
        raise ShapeError(f"importance mask shape {tuple(b_top.shape)} != {shape}")
    if tuple(cond.shape) != (layout.M_total, layout.M_total):
        raise ShapeError(f"condition mask shape {tuple(cond.shape)} is inconsistent with the layout")
    if tuple(adja.shape) != (layout.M_v, layout.M_v):
        raise ShapeError(f"adjacency mask shape {tuple(adja.shape)} is inconsistent with the layout")
    top = _dev.as_cuda(b_top)
    dense = top.to(torch.bool) | _dev.as_cuda(cond).to(torch.bool)[None, : layout.M_v, :]
    dense[:, :, : layout.M_v] |= _dev.as_cuda(adja).to(torch.bool)[None]
    return BlockMask(bits=dense, host=_dev.is_numpy(b_top))


def build_block_mask(q, k, layout: BlockLayout, statics: StaticMasks, params: SelectionParams,
                     *, need_relevance: bool = True):
    """Pool -> score -> select -> union; returns (BlockMask, R) (masks.py:178-199).

    With R (the reference's return value): pool, float64 scores into R, and the row-softmax +
    selection + union kernel that leaves R in place -- three launches.  ``need_relevance=False``
    (keyword extension; returns ``(mask, None)``) never materialises R: the scores go to a
    bounded scratch and, at p == 0, the selection runs on them directly (plus an exact re-run
    of near-tie rows) -- bitwise the same mask."""
    qd, kd = _poolable(q), _poolable(k)
    if qd.dtype != kd.dtype:
        qd, kd = qd.to(torch.float64), kd.to(torch.float64)
    _dev.same_device(qd, kd)
    with _dev.on(qd):
        return _build_block_mask(qd, kd, layout, statics, params, host=_dev.is_numpy(q),
                                 need_relevance=need_relevance)


def mask_buffers(H: int, layout: BlockLayout, device):
    """(bits, kv_cnt) device buffers of a mask with H heads."""
    words = mask_words(layout.M_total)
    return (torch.empty((H, layout.M_v, words), dtype=torch.int32, device=device),
            torch.empty((H, layout.M_v), dtype=torch.int32, device=device))


def mask_scratch(H: int, layout: BlockLayout, device) -> torch.Tensor:
    """Score scratch of the R-free mask launch (all heads up to 256 MB, else a bounded chunk)."""
    n = _native.query("tcb_block_mask_scratch", H, layout.M_v, layout.M_total)
    return torch.empty(n, dtype=torch.float64, device=device)


def launch_mask(pq: torch.Tensor, pk: torch.Tensor, layout: BlockLayout, adja, params,
                bits: torch.Tensor, kv_cnt: torch.Tensor, stream: int, scratch: torch.Tensor) -> None:
    """Scores -> select -> union on pooled (H, M_total, d) float64 means, no R returned."""
    H, _, d = pq.shape
    _native.call("tcb_block_mask", pq.data_ptr(), pq.shape[1], pk.data_ptr(), H, layout.M_v,
                 layout.M_total, d, _native.ptr(adja), mask_words(layout.M_total),
                 params.n_floor(layout.M_v), float(params.p), bits.data_ptr(), kv_cnt.data_ptr(),
                 scratch.data_ptr(), scratch.numel(), stream)


def _build_block_mask(qd, kd, layout, statics, params, host, need_relevance=True):
    d_k = qd.shape[-1]
    H = qd.shape[0]
    pq, pk = _pool_one_or_two(qd, kd, layout)
    bits, kv_cnt = mask_buffers(H, layout, qd.device)
    adja = statics.packed(layout)
    if not need_relevance:
        launch_mask(pq.values, pk.values, layout, adja, params, bits, kv_cnt, _dev.stream(),
                    mask_scratch(H, layout, qd.device))
        R = None
    else:
        R = torch.empty((H, layout.M_v, layout.M_total), dtype=torch.float64, device=qd.device)
        _native.call("tcb_block_scores", pq.values.data_ptr(), layout.M_total,
                     pk.values.data_ptr(), H, layout.M_v, layout.M_total, d_k, R.data_ptr(),
                     _dev.stream())
        _native.call("tcb_block_select_scores", R.data_ptr(), H, layout.M_v, layout.M_total,
                     _native.ptr(adja), mask_words(layout.M_total), params.n_floor(layout.M_v),
                     float(params.p), 1, bits.data_ptr(), kv_cnt.data_ptr(), _dev.stream())
    mask = BlockMask(words=bits, kv_cnt=kv_cnt, M_total=layout.M_total, nonempty=True, host=host)
    if R is not None and host:
        R = R.cpu().numpy()
    return mask, R


def mask_stats(mask: BlockMask, R=None, p: float | None = None) -> dict:
    """masks.py:202-213."""
    stats = {"n_heads": mask.n_heads, "shape": list(mask.shape),
             "selected_fraction": mask.selected_fraction}
    if R is not None and p is not None:
        Rd = _dev.as_cuda(R, torch.float64)
        covered = (Rd * mask.bits_dev[:, :, : Rd.shape[-1]]).sum(dim=-1) > p
        stats["rows_meeting_cutoff"] = int(covered.sum().item())
        stats["rows_total"] = int(covered.numel())
    return stats

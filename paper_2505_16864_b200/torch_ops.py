"""PyTorch operator registration of the path (``torch.ops.tokencarve.*``).

A PyTorch DiT calls carved attention inside its own (possibly ``torch.compile``-d) forward;
registering the C-ABI launches as custom operators with fake (meta) implementations makes
them opaque graph nodes with known output shapes, so the surrounding model can be traced
without breaking the graph at every layer.  The ops launch the same sm_100a kernels on the
current stream as the ``tokencarve``-API functions:

* ``tokencarve::block_mask(q, k, adja_bits, m, M_v, M_total, n_valid, n_cond, n_floor, p)``
  -> (words, kv_cnt): pool -> scores/select/union (no R) (masks.py:178-199);
* ``tokencarve::carve(q, k, v, words, kv_cnt, m, M_v, M_total, n_valid, n_cond, beta)``
  -> out: block-sparse attention (attention.py:209-243).
"""

from __future__ import annotations

import torch

from . import _dev, _native
from .attention import launch_carve
from .errors import ShapeError
from .partition import mask_words

__all__ = ["block_mask", "carve"]


@torch.library.custom_op("tokencarve::block_mask", mutates_args=())
def block_mask(q: torch.Tensor, k: torch.Tensor, adja_bits: torch.Tensor, m: int, M_v: int,
               M_total: int, n_valid: int, n_cond: int, n_floor: int,
               p: float) -> tuple[torch.Tensor, torch.Tensor]:
    from .masks import mask_scratch, launch_mask, mask_buffers
    from .partition import BlockLayout

    H, _, d = q.shape
    dev = q.device
    lay = BlockLayout(m=m, n_valid=n_valid, n_cond=n_cond, M_v=M_v, M_c=M_total - M_v)
    with torch.cuda.device(dev):
        s = torch.cuda.current_stream(dev).cuda_stream
        pq = torch.empty((H, M_total, d), dtype=torch.float64, device=dev)
        pk = torch.empty_like(pq)
        bits, kv_cnt = mask_buffers(H, lay, dev)
        _native.call("tcb_block_pool", q.data_ptr(), k.data_ptr(), _dev.code_of(q.dtype),
                     q.stride(0), q.stride(1), H, d, m, M_v, M_total, n_valid, n_cond,
                     pq.data_ptr(), pk.data_ptr(), s)
        launch_mask(pq, pk, lay, adja_bits, _Floor(n_floor, p), bits, kv_cnt, s,
                    mask_scratch(H, lay, dev))
    return bits, kv_cnt


class _Floor:
    """SelectionParams stand-in carrying the host-computed n_floor (the op's argument)."""

    def __init__(self, n_floor: int, p: float):
        self._n, self.p = n_floor, p

    def n_floor(self, M_v: int) -> int:
        return self._n


@block_mask.register_fake
def _(q, k, adja_bits, m, M_v, M_total, n_valid, n_cond, n_floor, p):
    H = q.shape[0]
    words = mask_words(M_total)
    return (q.new_empty((H, M_v, words), dtype=torch.int32),
            q.new_empty((H, M_v), dtype=torch.int32))


@torch.library.custom_op("tokencarve::carve", mutates_args=())
def carve(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, bits: torch.Tensor,
          kv_cnt: torch.Tensor, m: int, M_v: int, M_total: int, n_valid: int, n_cond: int,
          beta: float) -> torch.Tensor:
    if not (q.dtype == k.dtype == v.dtype):
        raise ShapeError(f"q/k/v dtypes differ: {q.dtype}, {k.dtype}, {v.dtype}")
    if k.stride() != q.stride() or v.stride() != q.stride() or q.stride(2) != 1:
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    with torch.cuda.device(q.device):
        out = torch.empty_like(q)
        launch_carve(q, k, v, out, bits, kv_cnt, m, M_v, M_total, n_valid, n_cond, beta)
    return out


@carve.register_fake
def _(q, k, v, bits, kv_cnt, m, M_v, M_total, n_valid, n_cond, beta):
    return torch.empty_like(q)

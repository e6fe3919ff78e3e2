"""One carved-attention layer = ``build_block_mask`` + ``carve_attention``.

This is the pair of calls the reference's attention layer makes
(``toy_transformer_denoiser``, pipeline.py:432-433), exposed as one entry point so
that host-resident Q/K/V can be streamed through the GPU.  Carved attention is
independent per head (attention.py:236): pooling, scores, selection and
the sparse flash-attention of head h read only head h.  With host inputs the layer
therefore runs as a head-chunked pipeline on three CUDA streams --

    copy stream   H2D  q/k/v[chunk c+1]
    compute       pool -> scores/select (no R) -> carve on chunk c
    copy stream   D2H  out[chunk c-1]

-- so the PCIe transfers overlap the kernels and each other (PCIe is full duplex).
Each chunk's launches are the same kernels on head-slice views, so the result is
bitwise the unchunked one.  Device inputs take the plain two-call path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _native
from .attention import AmplifierBias, _workspace, carve_work_bytes
from .errors import ShapeError
from .masks import BlockMask, SelectionParams, mask_scratch, launch_mask, mask_buffers
from .partition import BlockLayout, StaticMasks

__all__ = ["carve_layer", "CarveLayerGraph"]

_streams: dict = {}


def _copy_streams(dev: torch.device):
    s = _streams.get(dev)
    if s is None:
        s = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        _streams[dev] = s
    return s


def _launch_chunk(q, k, v, o, pq, pk, bits, kv_cnt, scratch, adja, layout, params, beta, work,
                  sptr):
    """pool -> scores/select/union (no R) -> carve on head-slice views (H_c, N, d)."""
    Hc, _, d = q.shape
    sh, sn = q.stride(0), q.stride(1)
    Mv, Mt = layout.M_v, layout.M_total
    _native.call("tcb_block_pool", q.data_ptr(), k.data_ptr(), _dev.code_of(q.dtype), sh, sn, Hc, d,
                 layout.m, Mv, Mt, layout.n_valid, layout.n_cond, pq.data_ptr(), pk.data_ptr(), sptr)
    launch_mask(pq, pk, layout, adja, params, bits, kv_cnt, sptr, scratch)
    _native.call("tcb_carve_fwd", q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                 _dev.code_of(q.dtype), sh, sn, bits.data_ptr(), bits.shape[-1], kv_cnt.data_ptr(),
                 Hc, d, layout.m, Mv, Mt, layout.n_valid, layout.n_cond, float(beta), work.data_ptr(),
                 work.numel(), sptr)


def carve_layer(q, k, v, layout: BlockLayout, statics: StaticMasks, params: SelectionParams,
                beta: AmplifierBias = AmplifierBias(0.0), *, out=None,
                heads_per_chunk: int | None = None):
    """Carved attention for all heads; returns ``(out, BlockMask)``.

    q, k, v: (H, N_pad, d) bf16 or fp32, all three on the device or all three on the
    host (torch CPU tensors -- pinned for asynchronous copies -- or numpy arrays).
    Host inputs give a host output, complete on return (``out`` may supply a pinned
    (H, N_pad, d) tensor; numpy inputs return numpy); the returned mask stays on the device.
    """
    on_host = not (isinstance(q, torch.Tensor) and q.is_cuda)
    if not on_host:
        from .attention import AttentionInputs, carve_attention
        from .masks import build_block_mask

        mask, _ = build_block_mask(q, k, layout, statics, params, need_relevance=False)
        o = carve_attention(AttentionInputs(q=q, k=k, v=v, layout=layout), mask, beta)
        if out is not None:
            out.copy_(o)
            o = out
        return o, mask

    numpy_in = _dev.is_numpy(q)
    hq, hk, hv = (torch.from_numpy(np.ascontiguousarray(x)) if _dev.is_numpy(x) else x.contiguous()
                  for x in (q, k, v))
    if not (hq.shape == hk.shape == hv.shape) or hq.ndim != 3:
        raise ShapeError(f"Q/K/V must share one (heads, N, d_k) shape, got {tuple(hq.shape)}/"
                         f"{tuple(hk.shape)}/{tuple(hv.shape)}")
    if hq.shape[1] != layout.padded_total:
        raise ShapeError(f"token axis {hq.shape[1]} != padded token count {layout.padded_total}")
    if hq.dtype not in (torch.float32, torch.bfloat16) or hk.dtype != hq.dtype or hv.dtype != hq.dtype:
        raise ShapeError(f"Q/K/V must all be float32 or all bfloat16, got {hq.dtype}")
    H, N, d = hq.shape
    dev = _dev.device()
    if out is None:
        out = torch.empty((H, N, d), dtype=hq.dtype, pin_memory=True)
    elif tuple(out.shape) != (H, N, d) or out.dtype != hq.dtype or out.is_cuda:
        raise ShapeError("out must be a host tensor of the input shape and dtype")
    Mt = layout.M_total
    dq, dk, dv = (torch.empty((H, N, d), dtype=hq.dtype, device=dev) for _ in range(3))
    do = torch.empty((H, N, d), dtype=hq.dtype, device=dev)
    pq = torch.empty((H, Mt, d), dtype=torch.float64, device=dev)
    pk = torch.empty_like(pq)
    bits, kv_cnt = mask_buffers(H, layout, dev)
    scratch = mask_scratch(H, layout, dev)
    adja = statics.packed(layout)
    hc = heads_per_chunk or max(1, H // 12)  # C2: 2-head chunks (44.6 vs 45.2 ms at 3)
    work = _workspace(dev, carve_work_bytes(min(hc, H), layout.M_v, Mt, layout.m, d))

    comp = torch.cuda.current_stream(dev)
    s_in, s_out = _copy_streams(dev)
    chunks = [(h0, min(H, h0 + hc)) for h0 in range(0, H, hc)]
    s_in.wait_stream(comp)  # device buffers may be recycled from work still queued on comp
    s_out.wait_stream(comp)
    for h0, h1 in chunks:
        with torch.cuda.stream(s_in):
            for src, dst in ((hq, dq), (hk, dk), (hv, dv)):
                dst[h0:h1].copy_(src[h0:h1], non_blocking=True)
        comp.wait_stream(s_in)
        sl = slice(h0, h1)
        _launch_chunk(dq[sl], dk[sl], dv[sl], do[sl], pq[sl], pk[sl], bits[sl], kv_cnt[sl], scratch,
                      adja, layout, params, beta.beta, work, comp.cuda_stream)
        s_out.wait_stream(comp)
        with torch.cuda.stream(s_out):
            out[h0:h1].copy_(do[h0:h1], non_blocking=True)
    comp.wait_stream(s_out)
    for t in (dq, dk, dv, do, pq, pk):  # keep the caching allocator from recycling early
        t.record_stream(s_in)
        t.record_stream(s_out)
    mask = BlockMask(words=bits, kv_cnt=kv_cnt, M_total=Mt, nonempty=True)
    comp.synchronize()  # a host result is complete on return, like the reference's arrays
    return (out.numpy() if numpy_in else out), mask


class CarveLayerGraph:
    """One carved-attention layer captured as a CUDA graph on fixed device buffers.

    A DiT runs the same layer geometry every step, so the launches
    (pool -> scores/select/union (no R) -> carve) and the carve kernel's work-counter reset are
    recorded once and replayed with one ``cudaGraphLaunch``.  Like ``torch.cuda.CUDAGraph``
    the buffers are static: write the step's Q/K/V into ``q``/``k``/``v`` (or pass the
    tensors the caller already fills in place), call :meth:`replay`, read ``out`` and
    ``mask``.  The replay is bitwise the eager ``carve_layer`` (same kernels, same order).
    """

    def __init__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: BlockLayout,
                 statics: StaticMasks, params: SelectionParams,
                 beta: AmplifierBias = AmplifierBias(0.0)):
        if not (isinstance(q, torch.Tensor) and q.is_cuda and k.is_cuda and v.is_cuda):
            raise ShapeError("CarveLayerGraph takes device Q/K/V (the static replay buffers)")
        if not (q.shape == k.shape == v.shape) or q.ndim != 3:
            raise ShapeError(f"Q/K/V must share one (heads, N, d_k) shape, got {tuple(q.shape)}/"
                             f"{tuple(k.shape)}/{tuple(v.shape)}")
        if q.shape[1] != layout.padded_total:
            raise ShapeError(f"token axis {q.shape[1]} != padded token count {layout.padded_total}")
        if k.stride() != q.stride() or v.stride() != q.stride() or q.stride(2) != 1:
            raise ShapeError("Q/K/V must share strides with a contiguous innermost axis")
        H, N, d = q.shape
        dev = q.device
        Mt = layout.M_total
        self.q, self.k, self.v = q, k, v
        self.out = torch.empty_like(q)
        self._pq = torch.empty((H, Mt, d), dtype=torch.float64, device=dev)
        self._pk = torch.empty_like(self._pq)
        self._bits, self._kv_cnt = mask_buffers(H, layout, dev)
        self._scratch = mask_scratch(H, layout, dev)
        self._adja = statics.packed(layout)
        # private (replays may overlap): counter + split condition-row partials
        self._work = torch.zeros(carve_work_bytes(H, layout.M_v, Mt, layout.m, d), dtype=torch.uint8,
                                 device=dev)
        self.mask = BlockMask(words=self._bits, kv_cnt=self._kv_cnt, M_total=Mt, nonempty=True)
        args = (self.q, self.k, self.v, self.out, self._pq, self._pk, self._bits, self._kv_cnt,
                self._scratch, self._adja, layout, params, beta.beta, self._work)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # eager warm-up: kernel attributes, tensor-map driver entry
            _launch_chunk(*args, side.cuda_stream)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            _launch_chunk(*args, torch.cuda.current_stream(dev).cuda_stream)

    def replay(self) -> torch.Tensor:
        """Run the captured layer on the current stream; returns ``out``."""
        self.graph.replay()
        return self.out

"""Head-parallel carved attention across G GPUs (Ulysses-style all-to-all).

Outside attention each rank holds a contiguous curve-order token shard (N_pad/G tokens, all
H heads) -- the paper splits tokens by SFC index.  Carved attention is
independent per head (attention.py:236), so one all-to-all turns the sequence
shard into a head shard (all N_pad tokens, H/G heads), each rank runs pool -> select ->
carve locally on its heads, and a second all-to-all returns O to the token shard.

Exchange layout (zero repacking).  A rank's token shard is held as
``(C, G, n_loc, hc, d)``: chunk c (of C head chunks), destination rank g, local token t,
head j of that rank's chunk -- i.e. head ``g*H/G + c*hc + j`` of token t.  Then

* chunk c's send buffer for ``all_to_all_single`` is the contiguous slab ``x[c]``
  (no ``permute().contiguous()`` before the collective);
* what arrives, ``(G, n_loc, hc, d)``, *is* the token-major head shard ``(N_pad, hc, d)``
  (token-ordered because ranks hold consecutive token ranges), consumed in place by the
  pool / select / carve kernels through their (stride_h, stride_n) arguments;
* the carve kernel writes O straight into the next send buffer in that same token-major
  layout, and the return all-to-all lands it in the output shard's ``(C, G, n_loc, hc, d)``
  slab -- the layout the input came in, so consecutive layers never repack.

``to_exchange_layout`` converts an ``(n_loc, H, d)`` shard once (one copy), and
``from_exchange_layout`` gives the ``(n_loc, H, d)`` view back (a copy only if the caller
asks for contiguity).  ``chunks > 1`` pipelines the exchange: the (async, NCCL) all-to-all
of chunk c+1 runs while chunk c computes, and chunk c's output exchange runs under chunk
c+1's compute; carved attention is per-head, so the result is bitwise the unchunked one.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .partition import BlockLayout

__all__ = ["to_exchange_layout", "from_exchange_layout", "default_chunks", "seq_to_head",
           "head_to_seq", "carve_layer_sp", "carve_layer_sp_chunked"]


def default_chunks(heads_per_rank: int) -> int:
    """Head chunks of the pipelined exchange: the smallest divisor >= 2 of the rank's head
    count (C2 / 24 heads: 2 chunks at G = 2 and 4, 3 single-head chunks at G = 8; C3 / 40
    heads: 5 at G = 8), so the next chunk's collective always overlaps this chunk's compute;
    1 for a single head."""
    for c in range(2, heads_per_rank + 1):
        if heads_per_rank % c == 0:
            return c
    return 1


def to_exchange_layout(x: torch.Tensor, G: int, chunks: int = 1) -> torch.Tensor:
    """(n_loc, H, d) token shard -> (C, G, n_loc, hc, d) exchange layout (one copy)."""
    n_loc, H, d = x.shape
    if H % (G * chunks):
        raise ValueError(f"heads {H} not divisible by world size {G} x {chunks} chunks")
    hc = H // (G * chunks)
    return x.view(n_loc, G, chunks, hc, d).permute(2, 1, 0, 3, 4).contiguous()


def from_exchange_layout(xe: torch.Tensor, contiguous: bool = False) -> torch.Tensor:
    """(C, G, n_loc, hc, d) -> the (n_loc, H, d) token shard (a strided view unless
    ``contiguous``; heads ordered g*H/G + c*hc + j)."""
    C, G, n_loc, hc, d = xe.shape
    v = xe.permute(2, 1, 0, 3, 4)  # (n_loc, G, C, hc, d)
    return v.reshape(n_loc, G * C * hc, d) if contiguous else v


def _all_to_all(recv: torch.Tensor, send: torch.Tensor, group=None) -> None:
    """NCCL all_to_all_single over NVLink; a gloo group (CPU tests, or several ranks
    sharing one GPU in the orchestration test) stages CUDA tensors through the host."""
    if recv.is_cuda and dist.get_backend(group) == "gloo":
        r = torch.empty(recv.shape, dtype=recv.dtype)
        dist.all_to_all_single(r, send.cpu(), group=group)
        recv.copy_(r)
        return
    dist.all_to_all_single(recv, send, group=group)


def _a2a_async(recv: torch.Tensor, send: torch.Tensor, group=None):
    """Asynchronous all-to-all (NCCL runs it on its own stream; the returned work's
    ``wait()`` makes the current stream wait).  gloo stages through the host, synchronously."""
    if recv.is_cuda and dist.get_backend(group) == "gloo":
        _all_to_all(recv, send, group)
        return None
    return dist.all_to_all_single(recv, send, group=group, async_op=True)


def _exchange_input(x: torch.Tensor, G: int, chunks: int) -> torch.Tensor:
    """Accept a (C, G, n_loc, hc, d) exchange-layout tensor as is, or pack an (n_loc, H, d)
    shard (the only copy on the input side)."""
    if x.ndim == 5:
        if x.shape[0] != chunks or x.shape[1] != G or not x.is_contiguous():
            raise ValueError(f"exchange-layout input must be contiguous ({chunks}, {G}, n_loc, hc, d)")
        return x
    return to_exchange_layout(x, G, chunks)


def seq_to_head(xs: list, group=None) -> list:
    """[(N/G, H, d) or (1, G, N/G, H/G, d)] -> [(N, H/G, d)] token-major head shards."""
    G = dist.get_world_size(group)
    outs = []
    for x in xs:
        send = _exchange_input(x, G, 1)[0]  # (G, n_loc, hg, d): slab g goes to rank g
        recv = torch.empty_like(send)
        _all_to_all(recv, send, group)
        outs.append(recv.view(-1, send.shape[2], send.shape[3]))
    return outs


def head_to_seq(o: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """(N, H/G, d) contiguous token-major head shard -> the output shard in exchange layout
    (1, G, N/G, H/G, d) (view it with ``from_exchange_layout``); no repack either side."""
    G = dist.get_world_size(group)
    N, hg, d = o.shape
    send = o.view(G, N // G, hg, d)  # the carve output buffer is the send buffer
    recv = out[0] if out is not None else torch.empty_like(send)
    _all_to_all(recv, send, group)
    return recv.unsqueeze(0) if out is None else out


def carve_layer_sp(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: BlockLayout,
                   local_fn: Callable, group=None, chunks: int | None = 1) -> torch.Tensor:
    """Sequence-sharded q/k/v -> sequence-sharded output in exchange layout.

    q/k/v: (n_loc, H, d) token shards (packed once) or (C, G, n_loc, hc, d) exchange-layout
    tensors (zero copy).  ``local_fn(qh, kh, vh, layout, out=oh)`` receives head-major
    *views* (hc, N, d) of the token-major head shards and writes its result into ``oh``
    (same strides), the buffer the return all-to-all sends from.  ``chunks=None`` picks
    :func:`default_chunks`.  Returns (C, G, n_loc, hc, d); :func:`from_exchange_layout` views
    it as (n_loc, H, d)."""
    G = dist.get_world_size(group)
    H = q.shape[0] * q.shape[1] * q.shape[3] if q.ndim == 5 else q.shape[1]
    hg = H // G
    if chunks is None:
        chunks = q.shape[0] if q.ndim == 5 else default_chunks(hg)
    if chunks == 1:
        qe, ke, ve = (_exchange_input(x, G, 1) for x in (q, k, v))
        ins = []
        for x in (qe, ke, ve):
            recv = torch.empty_like(x[0])
            _all_to_all(recv, x[0], group)
            ins.append(recv)
        n_loc, d = qe.shape[2], qe.shape[4]
        views = [t.view(G * n_loc, hg, d).permute(1, 0, 2) for t in ins]  # (hg, N, d)
        oh = torch.empty((G * n_loc, hg, d), dtype=qe.dtype, device=qe.device)
        local_fn(*views, layout, out=oh.permute(1, 0, 2))
        out = torch.empty_like(qe)
        head_to_seq(oh, group, out=out)
        return out
    return carve_layer_sp_chunked(q, k, v, layout, local_fn, chunks=chunks, group=group)


def carve_layer_sp_chunked(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: BlockLayout,
                           local_fn: Callable, chunks: int = 2, group=None) -> torch.Tensor:
    """``carve_layer_sp`` with the exchange pipelined over head chunks (see the module doc);
    bitwise the unchunked result.  Returns (C, G, n_loc, hc, d)."""
    G = dist.get_world_size(group)
    if q.ndim == 5:
        chunks = q.shape[0]
    else:
        hg = q.shape[1] // G
        chunks = max(1, min(chunks, hg))
        if hg % chunks:
            raise ValueError(f"{hg} heads per rank not divisible into {chunks} chunks")
    qe, ke, ve = (_exchange_input(x, G, chunks) for x in (q, k, v))
    _, _, n_loc, hc, d = qe.shape

    def post_in(c):
        ins, works = [], []
        for x in (qe, ke, ve):
            recv = torch.empty_like(x[c])  # (G, n_loc, hc, d) == token-major (N, hc, d)
            works.append(_a2a_async(recv, x[c], group))
            ins.append(recv)
        return ins, works

    out = torch.empty_like(qe)
    pending = post_in(0)
    sends = []
    for c in range(chunks):
        ins, works = pending
        if c + 1 < chunks:
            pending = post_in(c + 1)  # exchange of the next chunk overlaps this compute
        for w in works:
            if w is not None:
                w.wait()
        views = [t.view(G * n_loc, hc, d).permute(1, 0, 2) for t in ins]  # (hc, N, d)
        oh = torch.empty((G * n_loc, hc, d), dtype=qe.dtype, device=qe.device)
        local_fn(*views, layout, out=oh.permute(1, 0, 2))
        sends.append((oh, _a2a_async(out[c], oh.view(G, n_loc, hc, d), group)))
    for oh, w in sends:  # keep the send buffers alive until their collectives complete
        if w is not None:
            w.wait()
    return out

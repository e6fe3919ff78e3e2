"""Head-parallel carved attention across G GPUs (Ulysses-style all-to-all).

Outside attention each rank holds a contiguous curve-order token shard
(N_pad/G tokens, all H heads) -- the paper splits tokens by SFC index
(PAPER.md:633-635).  Carved attention is independent per head (SPEC.md:208,
attention.py:236), so one all-to-all turns the sequence shard into a head shard
(all N_pad tokens, H/G heads), each rank runs pool -> select -> carve locally on
its heads, and a second all-to-all returns O to the token shard.

The head-sharded tensors are consumed in place as (N, H/G, d) token-major
buffers: the kernels take (stride_h, stride_n) so no transpose copy is needed
between the collective and the kernels.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .partition import BlockLayout

__all__ = ["seq_to_head", "head_to_seq", "carve_layer_sp", "carve_layer_sp_chunked"]


def _all_to_all(recv: torch.Tensor, send: torch.Tensor, group=None) -> None:
    """NCCL all_to_all_single over NVLink; a gloo group (CPU tests, or several ranks
    sharing one GPU in the orchestration test) stages CUDA tensors through the host."""
    if recv.is_cuda and dist.get_backend(group) == "gloo":
        r = torch.empty(recv.shape, dtype=recv.dtype)
        dist.all_to_all_single(r, send.cpu(), group=group)
        recv.copy_(r)
        return
    dist.all_to_all_single(recv, send, group=group)


def seq_to_head(xs: list, group=None) -> list:
    """[(N/G, H, d)] per tensor -> [(N, H/G, d)] head shards, one collective for all."""
    G = dist.get_world_size(group)
    n_loc, H, d = xs[0].shape
    if H % G:
        raise ValueError(f"heads {H} not divisible by world size {G}")
    hg = H // G
    outs = []
    for x in xs:
        # send[r] = our tokens of rank r's heads; recv[r] = rank r's tokens of our heads,
        # so recv viewed as (G*n_loc, hg, d) is already the token-ordered head shard
        send = x.view(n_loc, G, hg, d).permute(1, 0, 2, 3).contiguous()
        recv = torch.empty_like(send)
        _all_to_all(recv, send, group)
        outs.append(recv.view(G * n_loc, hg, d))
    return outs


def head_to_seq(o: torch.Tensor, group=None) -> torch.Tensor:
    """(N, H/G, d) head shard -> (N/G, H, d) token shard."""
    G = dist.get_world_size(group)
    N, hg, d = o.shape
    n_loc = N // G
    send = o.contiguous().view(G, n_loc, hg, d)
    recv = torch.empty_like(send)
    _all_to_all(recv, send, group)
    return recv.permute(1, 0, 2, 3).reshape(n_loc, G * hg, d)


def carve_layer_sp(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: BlockLayout,
                   local_fn: Callable, group=None) -> torch.Tensor:
    """Sequence-sharded (N/G, H, d) q/k/v -> sequence-sharded output.

    ``local_fn(qh, kh, vh, layout)`` receives head-major *views* (H/G, N, d) of the
    token-major head shards and returns the output in the same form.
    """
    qh, kh, vh = seq_to_head([q, k, v], group)
    views = [t.permute(1, 0, 2) for t in (qh, kh, vh)]  # (H/G, N, d), stride (d, H/G*d, 1)
    oh = local_fn(*views, layout)
    return head_to_seq(oh.permute(1, 0, 2), group)


def _a2a_async(recv: torch.Tensor, send: torch.Tensor, group=None):
    """Asynchronous all-to-all (NCCL runs it on its own stream; the returned work's
    ``wait()`` makes the current stream wait).  gloo stages through the host, synchronously."""
    if recv.is_cuda and dist.get_backend(group) == "gloo":
        _all_to_all(recv, send, group)
        return None
    return dist.all_to_all_single(recv, send, group=group, async_op=True)


def carve_layer_sp_chunked(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: BlockLayout,
                           local_fn: Callable, chunks: int = 2, group=None) -> torch.Tensor:
    """``carve_layer_sp`` with the exchange pipelined over head chunks: the all-to-all of
    chunk c+1 (NCCL, async) runs while chunk c is pooled / selected / carved, and chunk c's
    output all-to-all runs under chunk c+1's compute.  Each rank's H/G heads are split into
    ``chunks`` groups; chunk c carries heads [c*hc, (c+1)*hc) of every rank's slice.  Carved
    attention is independent per head, so the result equals the unchunked exchange
    bitwise."""
    G = dist.get_world_size(group)
    n_loc, H, d = q.shape
    if H % G:
        raise ValueError(f"heads {H} not divisible by world size {G}")
    hg = H // G
    chunks = max(1, min(chunks, hg))
    if hg % chunks:
        raise ValueError(f"{hg} heads per rank not divisible into {chunks} chunks")
    hc = hg // chunks

    def send_of(x, c):  # (G, n_loc, hc, d): for rank r, our tokens of its chunk-c heads
        return x.view(n_loc, G, hg, d)[:, :, c * hc:(c + 1) * hc].permute(1, 0, 2, 3).contiguous()

    def post_in(c):
        ins, works = [], []
        for x in (q, k, v):
            send = send_of(x, c)
            recv = torch.empty_like(send)
            works.append(_a2a_async(recv, send, group))
            ins.append(recv)
        return ins, works

    out = torch.empty_like(q)
    pending = post_in(0)
    outs = []
    for c in range(chunks):
        ins, works = pending
        if c + 1 < chunks:
            pending = post_in(c + 1)  # exchange of the next chunk overlaps this compute
        for w in works:
            if w is not None:
                w.wait()
        views = [t.view(G * n_loc, hc, d).permute(1, 0, 2) for t in ins]  # (hc, N, d)
        oh = local_fn(*views, layout)  # (hc, N, d) head-major view of a token-major shard
        send = oh.permute(1, 0, 2).contiguous().view(G, n_loc, hc, d)
        recv = torch.empty_like(send)
        outs.append((c, recv, _a2a_async(recv, send, group)))
    ov = out.view(n_loc, G, hg, d)
    for c, recv, w in outs:
        if w is not None:
            w.wait()
        ov[:, :, c * hc:(c + 1) * hc] = recv.permute(1, 0, 2, 3)
    return out

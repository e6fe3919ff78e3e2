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

__all__ = ["seq_to_head", "head_to_seq", "carve_layer_sp"]


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

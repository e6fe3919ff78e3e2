"""The Ulysses head-parallel layer with the REAL kernels, several ranks sharing cuda:0.

2 and 4 processes join a gloo group (the exchange is staged through the host -- the only
multi-rank transport a 1-GPU box offers; on a node the same code runs over NCCL), each
holds a curve-order token shard, and ``carve_layer_sp`` / the pipelined
``carve_layer_sp_chunked`` run build_block_mask (R-free path) + the tcgen05 carve kernel on
each rank's head shard, consumed in place as token-major (N, H/G, d) strided views and
written straight into the return exchange's send buffer.  The gathered output must equal
the single-rank layer bitwise (carved attention is independent per head, and neither kernel
depends on the strides).

A 1-GPU box cannot host two NCCL ranks (NCCL rejects two ranks on one device), so the NCCL
code path -- ``all_to_all_single`` on device tensors, its ``async_op`` works waited on the
compute stream in the pipelined exchange -- runs as a world of one: every collective is a
self-exchange, but the streams, waits and buffer lifetimes are the ones a node uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

DIMS, M, NC, H, D = (4, 16, 24), 128, 200, 8, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(tcb):
    g = tcb.GridDims(*DIMS)
    lay = tcb.build_layout(g, M, NC)
    st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
    gen = torch.Generator(device="cuda").manual_seed(99)
    q, k, v = (torch.randn((H, lay.padded_total, D), generator=gen, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    return lay, st, q, k, v


def _worker(rank, world, port, out_path, chunks, pre_layout, backend="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2505_16864_b200 as tcb
    from paper_2505_16864_b200.ulysses import (carve_layer_sp, carve_layer_sp_chunked,
                                               from_exchange_layout, to_exchange_layout)

    lay, st, q, k, v = _inputs(tcb)
    prm = tcb.SelectionParams(k=0.3, p=0.0)
    n_loc = lay.padded_total // world

    def shard(x):  # (H, N, d) -> this rank's token shard (N/G, H, d)
        return x.permute(1, 0, 2)[rank * n_loc:(rank + 1) * n_loc].contiguous()

    calls = []

    def local(qh, kh, vh, layout, out):
        assert qh.stride(2) == 1 and qh.stride(0) == D  # token-major head shard, in place
        mask, _ = tcb.build_block_mask(qh, kh, layout, st, prm, need_relevance=False)
        tcb.carve_raw(qh, kh, vh, mask, layout, 0.2, out=out)
        calls.append(qh.shape[0])

    xs = [shard(x) for x in (q, k, v)]
    if pre_layout:
        xs = [to_exchange_layout(x, world, chunks) for x in xs]
        o = carve_layer_sp(*xs, lay, local, chunks=None)
    elif chunks > 1:
        o = carve_layer_sp_chunked(*xs, lay, local, chunks=chunks)
    else:
        o = carve_layer_sp(*xs, lay, local)
    assert sum(calls) == H // world
    torch.save(from_exchange_layout(o, contiguous=True).cpu(), f"{out_path}.{rank}")
    dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks,pre_layout,backend", [
    (2, 1, False, "gloo"), (2, 2, False, "gloo"), (4, 1, False, "gloo"), (4, 2, False, "gloo"),
    (4, 2, True, "gloo"), (1, 1, False, "nccl"), (1, 2, False, "nccl"), (1, 4, True, "nccl")])
def test_ulysses_real_kernels_bitwise(tmp_path, world, chunks, pre_layout, backend):
    import paper_2505_16864_b200 as tcb

    lay, st, q, k, v = _inputs(tcb)
    assert lay.padded_total % world == 0
    mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=0.3, p=0.0))
    full = tcb.carve_raw(q, k, v, mask, lay, 0.2).permute(1, 0, 2).cpu()  # (N, H, d)
    out = str(tmp_path / "o")
    mp.spawn(_worker, args=(world, _free_port(), out, chunks, pre_layout, backend), nprocs=world,
             join=True)
    got = torch.cat([torch.load(f"{out}.{r}") for r in range(world)], dim=0)
    assert got.shape == full.shape
    assert torch.equal(got, full)

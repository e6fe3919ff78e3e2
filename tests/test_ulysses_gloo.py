"""World-size-2 gloo test (CPU) of the Ulysses sequence<->head exchange around a
per-head attention: sharded result == unsharded oracle result, for the packed (n_loc, H, d)
input, the pipelined exchange, and inputs already in the (C, G, n_loc, hc, d) exchange
layout."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(H=4):
    dims, m, nc, d = (2, 6, 8), 8, 5, 16
    L = oracle.layout_scalars(dims, m, nc)
    rng = np.random.default_rng(3)
    q, k, v = (rng.standard_normal((H, L["padded_total"], d)).astype(np.float32) for _ in range(3))
    inv = oracle.curve_inverse(oracle.curve_forward(dims))
    adja = oracle.adjacency(dims, inv, m, L["M_v"])
    return dims, L, q, k, v, adja


def _worker(rank, world, port, out_path, chunks=0, heads=4):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_16864_b200.ulysses import (carve_layer_sp, carve_layer_sp_chunked,
                                               from_exchange_layout, to_exchange_layout)

    dims, L, q, k, v, adja = _case(heads)
    N = L["padded_total"]
    n_loc = N // world

    def shard(x):  # (H, N, d) -> token shard (N/G, H, d)
        return torch.from_numpy(np.ascontiguousarray(x.transpose(1, 0, 2)[rank * n_loc:(rank + 1) * n_loc]))

    def local(qh, kh, vh, layout, out):
        # per-head layer on the head shard: mask build + carve (the exchange is what is tested
        # here; tests/test_gpu_ulysses.py runs the same exchange around the real kernels)
        qn, kn, vn = (t.contiguous().numpy() for t in (qh, kh, vh))
        bits, _ = oracle.block_mask(qn, kn, L, adja, 0.3, 0.3)
        out.copy_(torch.from_numpy(oracle.carve(qn, kn, vn, bits, L, 0.25)))

    if chunks == -1:  # inputs already in the exchange layout: no packing at all
        xs = [to_exchange_layout(shard(x), world, 2) for x in (q, k, v)]
        o = carve_layer_sp(*xs, None, local, chunks=None)
    elif chunks is None:  # default chunking (an odd head count per rank: single-head chunks)
        o = carve_layer_sp(shard(q), shard(k), shard(v), None, local, chunks=None)
    elif chunks:
        o = carve_layer_sp_chunked(shard(q), shard(k), shard(v), None, local, chunks=chunks)
    else:
        o = carve_layer_sp(shard(q), shard(k), shard(v), None, local)
    torch.save(from_exchange_layout(o, contiguous=True), f"{out_path}.{rank}")
    dist.destroy_process_group()


@pytest.mark.parametrize("chunks,heads", [(0, 4), (1, 4), (2, 4), (-1, 4), (None, 6)])
def test_ulysses_roundtrip_world2(tmp_path, chunks, heads):
    if not dist.is_gloo_available():
        pytest.skip("gloo missing")
    N_pad = _case(heads)[1]["padded_total"]
    assert N_pad % 2 == 0
    port = _free_port()
    out = str(tmp_path / "o")
    mp.spawn(_worker, args=(2, port, out, chunks, heads), nprocs=2, join=True)
    dims, L, q, k, v, adja = _case(heads)
    bits, _ = oracle.block_mask(q, k, L, adja, 0.3, 0.3)
    full = oracle.carve(q, k, v, bits, L, 0.25).transpose(1, 0, 2)  # (N, H, d)
    got = np.concatenate([torch.load(f"{out}.{r}").numpy() for r in range(2)], axis=0)
    np.testing.assert_array_equal(got, full)

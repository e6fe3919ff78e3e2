"""Loading helpers for the committed golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import functools
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name: str):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def small_curves():
    g = load("curves.npz")
    off = g["small_offsets"]
    for i, dims in enumerate(g["small_dims"]):
        yield tuple(int(v) for v in dims), g["small_forward"][off[i]:off[i + 1]]


def layout_rows():
    g = load("layouts.npz")
    off = g["adj_offsets"]
    for i, r in enumerate(g["rows"]):
        dims = tuple(int(v) for v in r[:3])
        m, nc = int(r[3]), int(r[4])
        M_v = int(r[6])
        adj = np.unpackbits(g["adj_packed"][off[i]:off[i + 1]])[: M_v * M_v].reshape(M_v, M_v)
        yield dims, m, nc, r, adj.astype(bool)


def qkv(seed, H, N, d):
    rng = np.random.default_rng(seed)
    return tuple(rng.standard_normal((H, N, d), dtype=np.float32) for _ in range(3))


def unpack_bits(packed, n_cols):
    return np.unpackbits(packed, axis=-1)[..., :n_cols].astype(bool)


def mask_cases():
    g = load("masks.npz")
    for name, meta in zip(g["names"], g["meta"]):
        t, h, w, m, nc, H, d, seed = (int(v) for v in meta[:8])
        k, p = float(meta[8]), float(meta[9])
        yield str(name), dict(dims=(t, h, w), m=m, n_cond=nc, H=H, d=d, seed=seed, k=k, p=p), g


def attention_cases():
    g = load("attention.npz")
    for name, meta in zip(g["names"], g["meta"]):
        t, h, w, m, nc, H, d, seed = (int(v) for v in meta[:8])
        k, p, beta = float(meta[8]), float(meta[9]), float(meta[10])
        yield str(name), dict(dims=(t, h, w), m=m, n_cond=nc, H=H, d=d, seed=seed, k=k, p=p,
                              beta=beta), g


def host(x):
    """numpy view of a result that is numpy (numpy callers) or a device tensor."""
    return x if isinstance(x, np.ndarray) else x.detach().cpu().numpy()

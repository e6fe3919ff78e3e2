"""numpy restatement of the reference ``tokencarve`` hot path.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Every function cites
the reference file:line (relative to ``/root/reference/pkg/src/tokencarve``)
whose behaviour it restates.  Nothing here is shared with the CUDA product
path; the restatement is pinned against golden vectors generated from the
real reference (``tests/golden``).

Conventions: arrays are numpy; integer permutations are int64 like the
reference; masks are dense bool (H, M_v, M_total).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "plane_order",
    "curve_forward",
    "curve_inverse",
    "layout_scalars",
    "token_valid",
    "block_counts",
    "adjacency",
    "condition",
    "pool_blocks",
    "relevance_f64",
    "select_topk",
    "union_bits",
    "block_mask",
    "carve",
    "dense_reference",
    "mask_to_bias",
    "area_weights",
    "upsample_area",
    "transition",
    "beta_of",
    "curve_positions",
    "patchify",
    "unpatchify",
    "rope_table",
    "rope_apply",
]


# --------------------------------------------------------------------------
# L1: space-filling curve (sfc.py)
# --------------------------------------------------------------------------

def plane_order(a: int, b: int) -> list:
    """Generalized-Hilbert visit order of an a x b plane from (0, 0).

    Restates ``_gilbert2d``/``_gen2d`` (sfc.py:98-157): the longer axis is the
    major axis; a rectangle splits in two along the major axis when
    ``2w > 3h`` (odd-half fix when ``w > 2``), otherwise in three
    (up / across / down, odd-half fix when ``h > 2``).  Python floor division
    on negative vectors is essential (sfc.py:133-134).
    """
    out = []

    def sgn(v):
        return (v > 0) - (v < 0)

    # explicit stack instead of recursion (same visit order)
    stack = [(0, 0, a, 0, 0, b) if a >= b else (0, 0, 0, b, a, 0)]
    while stack:
        x, y, ax, ay, bx, by = stack.pop()
        w, h = abs(ax + ay), abs(bx + by)
        ux, uy, vx, vy = sgn(ax), sgn(ay), sgn(bx), sgn(by)
        if h == 1:
            out.extend((x + i * ux, y + i * uy) for i in range(w))
            continue
        if w == 1:
            out.extend((x + i * vx, y + i * vy) for i in range(h))
            continue
        hax, hay, hbx, hby = ax // 2, ay // 2, bx // 2, by // 2
        if 2 * w > 3 * h:
            if abs(hax + hay) % 2 and w > 2:
                hax, hay = hax + ux, hay + uy
            children = [
                (x, y, hax, hay, bx, by),
                (x + hax, y + hay, ax - hax, ay - hay, bx, by),
            ]
        else:
            if abs(hbx + hby) % 2 and h > 2:
                hbx, hby = hbx + vx, hby + vy
            children = [
                (x, y, hbx, hby, hax, hay),
                (x + hbx, y + hby, ax, ay, bx - hbx, by - hby),
                (x + (ax - ux) + (hbx - vx), y + (ay - uy) + (hby - vy),
                 -hbx, -hby, -(ax - hax), -(ay - hay)),
            ]
        stack.extend(reversed(children))
    return out


def curve_forward(dims) -> np.ndarray:
    """Row-major cell id at every curve position (sfc.py:160-210).

    Shortest axis (ties: lowest index, ``np.argmin``) is swept in slice
    pairs; the plane order alternates forward/reversed per pair; within a
    pair the walk zig-zags between the two slices and the last plane cell
    always exits on the far slice (sfc.py:176-188); a trailing odd slice is
    walked once (sfc.py:190-193).
    """
    t, h, w = (int(v) for v in dims)
    shape = (t, h, w)
    s_ax = int(np.argmin(shape))
    p1, p2 = [a for a in range(3) if a != s_ax]
    plane = np.asarray(plane_order(shape[p1], shape[p2]), dtype=np.int64).reshape(-1, 2)
    n_plane = plane.shape[0]
    coords = np.empty((t * h * w, 3), dtype=np.int64)
    pos = 0
    pair = 0
    s = 0
    n_slab = shape[s_ax]
    while s < n_slab:
        seq = plane if pair % 2 == 0 else plane[::-1]
        if s + 1 < n_slab:
            i = np.arange(n_plane)
            first_lo = (i % 2 == 0) | (i == n_plane - 1)
            blk = np.empty((n_plane, 2, 3), dtype=np.int64)
            blk[:, :, p1] = seq[:, None, 0]
            blk[:, :, p2] = seq[:, None, 1]
            blk[:, 0, s_ax] = np.where(first_lo, s, s + 1)
            blk[:, 1, s_ax] = np.where(first_lo, s + 1, s)
            coords[pos:pos + 2 * n_plane] = blk.reshape(-1, 3)
            pos += 2 * n_plane
            s += 2
        else:
            blk = np.empty((n_plane, 3), dtype=np.int64)
            blk[:, p1] = seq[:, 0]
            blk[:, p2] = seq[:, 1]
            blk[:, s_ax] = s
            coords[pos:pos + n_plane] = blk
            pos += n_plane
            s += 1
        pair += 1
    return (coords[:, 0] * h + coords[:, 1]) * w + coords[:, 2]


def curve_inverse(forward: np.ndarray) -> np.ndarray:
    inv = np.empty_like(forward)
    inv[forward] = np.arange(forward.shape[0], dtype=forward.dtype)
    return inv


# --------------------------------------------------------------------------
# L2: block layout and static masks (partition.py)
# --------------------------------------------------------------------------

def layout_scalars(dims, m: int, n_cond: int = 0) -> dict:
    """Counts of ``build_layout`` (partition.py:91-104, sfc.py:240-251)."""
    n_valid = int(dims[0]) * int(dims[1]) * int(dims[2])
    M_v = -(-n_valid // m)
    M_c = -(-n_cond // m) if n_cond else 0
    return dict(m=m, n_valid=n_valid, n_cond=n_cond, M_v=M_v, M_c=M_c,
                M_total=M_v + M_c, cond_start=M_v * m, padded_total=(M_v + M_c) * m)


def token_valid(L: dict) -> np.ndarray:
    """partition.py:74-81: vision prefix and condition segment are valid."""
    ok = np.zeros(L["padded_total"], dtype=bool)
    ok[: L["n_valid"]] = True
    ok[L["cond_start"]: L["cond_start"] + L["n_cond"]] = True
    return ok


def block_counts(L: dict) -> np.ndarray:
    """partition.py:83-88."""
    return token_valid(L).reshape(L["M_total"], L["m"]).sum(axis=1)


def adjacency(dims, inverse: np.ndarray, m: int, M_v: int) -> np.ndarray:
    """26-neighbour block adjacency (partition.py:107-136).

    Every pair of Chebyshev-adjacent cells marks its two blocks; symmetric
    with a true diagonal.  Restated as: for each of the 13 lexicographically
    positive offsets, OR block(cell) x block(cell+offset).
    """
    t, h, w = (int(v) for v in dims)
    blk = (np.asarray(inverse) // m).reshape(t, h, w)
    A = np.eye(M_v, dtype=bool)
    for dt in (-1, 0, 1):
        for dh in (-1, 0, 1):
            for dw in (-1, 0, 1):
                if (dt, dh, dw) <= (0, 0, 0):
                    continue
                a = blk[max(dt, 0): t + min(dt, 0), max(dh, 0): h + min(dh, 0), max(dw, 0): w + min(dw, 0)]
                b = blk[max(-dt, 0): t + min(-dt, 0), max(-dh, 0): h + min(-dh, 0), max(-dw, 0): w + min(-dw, 0)]
                A[a.ravel(), b.ravel()] = True
    return A | A.T


def condition(M_v: int, M_total: int) -> np.ndarray:
    """partition.py:139-143: any row or column >= M_v."""
    c = np.arange(M_total) >= M_v
    return c[:, None] | c[None, :]


# --------------------------------------------------------------------------
# L3: dynamic block selection (masks.py)
# --------------------------------------------------------------------------

def pool_blocks(x: np.ndarray, L: dict):
    """Float64 mean over valid tokens per block (masks.py:98-116).

    Returns (values (H, M_total, d) float64, counts (M_total,)).  A block
    with no valid token pools to zeros.
    """
    H, N, d = x.shape
    ok = token_valid(L)
    z = np.where(ok[None, :, None], x, 0.0)
    s = z.reshape(H, L["M_total"], L["m"], d).sum(axis=2, dtype=np.float64)
    cnt = block_counts(L)
    return s / np.maximum(cnt, 1)[None, :, None], cnt


def relevance_f64(pq: np.ndarray, pk: np.ndarray, d_k: int) -> np.ndarray:
    """Row softmax of pooled scores / sqrt(d) in float64 (masks.py:119-134)."""
    s = np.matmul(pq, np.swapaxes(pk, 1, 2))
    s = s / math.sqrt(d_k)
    s = s - s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    return e / e.sum(axis=-1, keepdims=True)


def select_topk(R: np.ndarray, k: float, p: float, M_v: int) -> np.ndarray:
    """Importance selection (masks.py:137-159).

    Per row: descending stable order (ties -> lower column), sequential
    prefix sums, ``n_cut = #(prefix <= p) + 1``, floor ``max(1, ceil(k*M_v))``,
    cap at the column count; the first ``n_keep`` sorted columns are kept.
    """
    n_cols = R.shape[-1]
    order = np.argsort(-R, axis=-1, kind="stable")
    srt = np.take_along_axis(R, order, axis=-1)
    pre = np.cumsum(srt, axis=-1)
    n_cut = (pre <= p).sum(axis=-1) + 1
    floor_ = max(1, math.ceil(k * M_v))
    keep = np.minimum(np.maximum(n_cut, floor_), n_cols)
    sel = np.arange(n_cols) < keep[..., None]
    bits = np.zeros(R.shape, dtype=bool)
    np.put_along_axis(bits, order, sel, axis=-1)
    return bits


def union_bits(top: np.ndarray, adja: np.ndarray, M_v: int) -> np.ndarray:
    """masks.py:162-175: top | condition rows/cols | adjacency."""
    out = top.copy()
    out[:, :, M_v:] = True
    out[:, :, :M_v] |= adja[None]
    return out


def block_mask(q, k, L: dict, adja: np.ndarray, kk: float, p: float):
    """masks.py:178-199.  Returns (bits, R)."""
    d = q.shape[-1]
    pq, _ = pool_blocks(q, L)
    pk, _ = pool_blocks(k, L)
    R = relevance_f64(pq[:, : L["M_v"]], pk, d)
    top = select_topk(R, kk, p, L["M_v"])
    return union_bits(top, adja, L["M_v"]), R


# --------------------------------------------------------------------------
# L4: block-sparse attention (attention.py)
# --------------------------------------------------------------------------

def beta_of(numel_s: int, numel_S: int, rho: float) -> float:
    """attention.py:89-96."""
    return -rho * math.log(numel_s / numel_S) + 0.0


def _carve_one(q, k, v, bits, L, ok, beta, h, qb, out):
    """One (head, q-block) item, streaming softmax (attention.py:162-206)."""
    m = L["m"]
    d = q.shape[-1]
    sc = np.float32(1.0 / math.sqrt(d))
    vis = qb < L["M_v"]
    blocks = np.flatnonzero(bits[h, qb]) if vis else np.arange(L["M_total"])
    r = slice(qb * m, (qb + 1) * m)
    qs = q[h, r].astype(np.float32) * sc
    mx = np.full(m, -np.inf, np.float32)
    den = np.zeros(m, np.float32)
    acc = np.zeros((m, d), np.float32)
    for b in blocks:
        c = slice(b * m, (b + 1) * m)
        lg = qs @ k[h, c].astype(np.float32).T
        lg = np.where(ok[c][None, :], lg, np.float32(-np.inf))
        if vis and beta and b >= L["M_v"]:
            lg = lg + np.float32(beta)
        nm = np.maximum(mx, lg.max(axis=1))
        al = np.exp(mx - nm, dtype=np.float32)
        pr = np.exp(lg - nm[:, None], dtype=np.float32)
        den = den * al + pr.sum(axis=1, dtype=np.float32)
        acc = acc * al[:, None] + pr @ v[h, c].astype(np.float32)
        mx = nm
    res = acc / den[:, None]
    res[~ok[r]] = 0.0
    out[h, r] = res


def carve(q, k, v, bits, L: dict, beta: float = 0.0, workers: int | None = None,
          items=None) -> np.ndarray:
    """Block-sparse attention, fp32 (attention.py:209-243).

    ``items`` optionally restricts the (head, q-block) work list (used for a
    bounded CPU-baseline sample); untouched rows stay zero.
    """
    H = q.shape[0]
    ok = token_valid(L)
    out = np.zeros(q.shape, dtype=np.float32)
    if items is None:
        items = [(h, b) for h in range(H) for b in range(L["M_total"])]
    if workers is None:
        workers = int(os.environ.get("TOKENCARVE_THREADS", "1"))
    if workers > 1:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(lambda it: _carve_one(q, k, v, bits, L, ok, beta, it[0], it[1], out), items))
    else:
        for h, b in items:
            _carve_one(q, k, v, bits, L, ok, beta, h, b, out)
    return out


def mask_to_bias(bits: np.ndarray, L: dict, beta: float = 0.0) -> np.ndarray:
    """Token-level additive bias (attention.py:145-159)."""
    H = bits.shape[0]
    m, Mv, Mt = L["m"], L["M_v"], L["M_total"]
    bb = np.zeros((H, Mt, Mt), np.float32)
    bb[:, :Mv, :] = np.where(bits, np.float32(0), np.float32(-np.inf))
    if beta:
        bb[:, :Mv, Mv:] += np.float32(beta)
    return np.repeat(np.repeat(bb, m, axis=1), m, axis=2)


def dense_reference(q, k, v, bias=None, valid=None) -> np.ndarray:
    """Two-pass dense softmax attention in fp32 (attention.py:112-142)."""
    H, N, d = q.shape
    ok = np.ones(N, bool) if valid is None else np.asarray(valid, bool)
    sc = np.float32(1.0 / math.sqrt(d))
    lg = (q.astype(np.float32) * sc) @ np.swapaxes(k.astype(np.float32), 1, 2)
    if bias is not None:
        lg = lg + bias.astype(np.float32)
    lg = np.where(ok[None, None, :], lg, np.float32(-np.inf))
    lg = lg - lg.max(axis=-1, keepdims=True)
    wt = np.exp(lg, dtype=np.float32)
    wt /= wt.sum(axis=-1, keepdims=True)
    o = wt @ v.astype(np.float32)
    o[:, ~ok, :] = 0.0
    return o


# --------------------------------------------------------------------------
# L5: progressive-resolution stage switch (pipeline.py)
# --------------------------------------------------------------------------

def area_weights(src: int, dst: int) -> np.ndarray:
    """(dst, src) overlap weights / step (pipeline.py:140-150)."""
    step = src / dst
    W = np.zeros((dst, src), np.float64)
    for o in range(dst):
        lo, hi = o * step, (o + 1) * step
        for i in range(int(math.floor(lo)), min(int(math.ceil(hi)), src)):
            W[o, i] = max(0.0, min(hi, i + 1) - max(lo, i))
    return W / step


def upsample_area(x: np.ndarray, target) -> np.ndarray:
    """Separable float64 area upsample, axis 0 -> 1 -> 2 (pipeline.py:153-173)."""
    src = x.shape[:3]
    dst = tuple(int(v) for v in target)
    if src == dst:
        return x.copy()
    y = x.astype(np.float64)
    for ax in range(3):
        if src[ax] != dst[ax]:
            y = np.moveaxis(np.tensordot(area_weights(src[ax], dst[ax]), y, axes=(1, ax)), 0, ax)
    return y.astype(x.dtype)


def transition(x0: np.ndarray, sigma: float, target, noise: np.ndarray) -> np.ndarray:
    """Re-noised switch with caller-supplied noise (pipeline.py:176-194)."""
    if sigma == 0.0:
        return upsample_area(x0, target)
    if sigma == 1.0:
        return noise
    up = upsample_area(x0, target).astype(np.float32)
    s = np.float32(sigma)
    return (np.float32(1.0) - s) * up + s * noise


# --------------------------------------------------------------------------
# §8f-1: neighbours of the path (positions, patchify, RoPE)
# --------------------------------------------------------------------------

def curve_positions(dims) -> np.ndarray:
    """apply_permutation(unravel_index(arange(n), dims), perm) (pipeline.py:334-337)."""
    t, h, w = (int(v) for v in dims)
    coords = np.stack(np.unravel_index(np.arange(t * h * w), (t, h, w)), axis=1).astype(np.int64)
    return coords[curve_forward(dims)]


def patchify(x: np.ndarray, dims, patch) -> np.ndarray:
    """(t*pt, h*ph, w*pw, C) -> (n, pt*ph*pw*C) tokens in row-major cell order, features
    ordered (pt, ph, pw, C).  Patch (1,1,1) is x.reshape(n, C) (pipeline.py:345)."""
    t, h, w = (int(v) for v in dims)
    pt, ph, pw = (int(v) for v in patch)
    C = x.shape[-1]
    y = x.reshape(t, pt, h, ph, w, pw, C).transpose(0, 2, 4, 1, 3, 5, 6)
    return np.ascontiguousarray(y.reshape(t * h * w, pt * ph * pw * C))


def unpatchify(tok: np.ndarray, dims, patch, C: int) -> np.ndarray:
    """Inverse of ``patchify``."""
    t, h, w = (int(v) for v in dims)
    pt, ph, pw = (int(v) for v in patch)
    y = tok.reshape(t, h, w, pt, ph, pw, C).transpose(0, 3, 1, 4, 2, 5, 6)
    return np.ascontiguousarray(y.reshape(t * pt, h * ph, w * pw, C))


def rope_table(dims, sections, theta: float) -> list:
    """Per axis (cos, sin) float32 tables (n_pos, d_a/2): angle pos * theta^(-2j/d_a) in
    float64.  Not in the reference (it has no positional embedding in attention); this is
    the 3D RoPE convention the fused kernel implements (HunyuanVideo sections 16/56/56)."""
    out = []
    for n_pos, da in zip((int(v) for v in dims), sections):
        inv = theta ** (-(np.arange(0, da, 2, dtype=np.float64)) / da)
        ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
        out.append((np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)))
    return out


def rope_apply(x: np.ndarray, pos: np.ndarray, sections, theta: float, dims) -> np.ndarray:
    """x (n, H, d) float32, pos (n, 3) -> rotated float32; pair (2j, 2j+1) of section a:
    (x0*c - x1*s, x0*s + x1*c), every product and sum rounded to float32."""
    tabs = rope_table(dims, sections, theta)
    out = x.copy()
    off = 0
    for a, da in enumerate(sections):
        if da == 0:
            continue
        c, s = tabs[a]
        cc = c[pos[:, a]][:, None, :]  # (n, 1, da/2)
        ss = s[pos[:, a]][:, None, :]
        x0 = x[:, :, off: off + da: 2]
        x1 = x[:, :, off + 1: off + da: 2]
        out[:, :, off: off + da: 2] = (x0 * cc).astype(np.float32) - (x1 * ss).astype(np.float32)
        out[:, :, off + 1: off + da: 2] = (x0 * ss).astype(np.float32) + (x1 * cc).astype(np.float32)
        off += da
    return out

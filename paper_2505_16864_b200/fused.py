"""Fused neighbours of the carved-attention path.

The reference's DiT loop (pipeline.py:331-371) permutes the positional metadata once per
stage, gathers the latent into curve order before every denoiser call and scatters the
velocity back before the Euler update / stage switch.  A real video DiT additionally
patchifies the latent and applies 3D rotary embeddings to Q/K before attention.  These
kernels do each of those neighbouring passes fused with the SFC permutation:

* ``curve_positions``   -- positions in curve order straight from ``perm.forward``
                           (== ``apply_permutation(unravel(arange(n)), perm)``, bitwise);
* ``patchify_permute``  -- latent -> curve-order tokens (patch 1x1x1 ==
                           ``apply_permutation(x.reshape(n, C), perm)``, bitwise);
* ``unpermute_euler``   -- ``denoise_step(x, invert_permutation(vel_curve), ...)`` in one
                           pass (bitwise the two-pass result);
* ``switch_stage_curve``-- ``switch_stage`` reading a curve-order velocity;
* ``rope_permute`` / ``qkv_to_curve`` -- raster token-major Q/K/V -> curve-order
                           head-major (H, N_pad, d) buffers with 3D RoPE on Q and K: one
                           read and one write per element.

The 3D RoPE convention (not part of the reference, which has no positional embedding in
attention): head dim split into (d_t, d_h, d_w) sections (HunyuanVideo: 16, 56, 56;
theta 256); in section a, pair j rotates elements (2j, 2j+1) by pos_a * theta^(-2j/d_a);
angles and cos/sin in float64 on the host, rounded to float32; rotation in float32.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _dev, _native
from .errors import DomainError, ShapeError
from .partition import BlockLayout
from .pipeline import _check_up, _noise_source, predict_clean, stage_transition, upsample_area_3d
from .sfc import GridDims, Permutation

__all__ = ["curve_positions", "patchify_permute", "unpermute_euler", "switch_stage_curve",
           "rope_tables", "rope_permute", "qkv_to_curve"]


def _check_perm(perm: Permutation, dims: GridDims):
    if perm.dims.as_tuple() != dims.as_tuple():
        raise ShapeError(f"permutation dims {perm.dims.as_tuple()} != token grid {dims.as_tuple()}")


def curve_positions(perm: Permutation) -> torch.Tensor:
    """(n, 3) int64 (t, h, w) of each curve position (pipeline.py:334-337)."""
    d = perm.dims
    n = d.n_cells
    pos = torch.empty((n, 3), dtype=torch.int64, device=perm.forward_dev.device)
    _native.call("tcb_curve_positions", perm.forward_dev.data_ptr(), n, d.t, d.h, d.w, pos.data_ptr(),
                 _dev.stream())
    return pos


def _patch_dims(x: torch.Tensor, dims: GridDims, patch):
    pt, ph, pw = (int(v) for v in patch)
    if x.ndim != 4:
        raise ShapeError(f"latent must be rank 4 (T, H, W, C), got shape {tuple(x.shape)}")
    want = (dims.t * pt, dims.h * ph, dims.w * pw)
    if tuple(int(v) for v in x.shape[:3]) != want:
        raise ShapeError(f"latent {tuple(x.shape[:3])} != token grid {dims.as_tuple()} x patch {patch}")
    return pt, ph, pw, int(x.shape[3])


def patchify_permute(x, perm: Permutation, patch=(1, 1, 1)) -> torch.Tensor:
    """Latent (t*pt, h*ph, w*pw, C) float32 -> curve-order tokens (n, pt*ph*pw*C)."""
    xt = _dev.as_cuda(x).float().contiguous()
    dims = perm.dims
    pt, ph, pw, C = _patch_dims(xt, dims, patch)
    tok = torch.empty((dims.n_cells, pt * ph * pw * C), dtype=torch.float32, device=xt.device)
    _native.call("tcb_patchify_permute", xt.data_ptr(), perm.forward_dev.data_ptr(), dims.t, dims.h,
                 dims.w, pt, ph, pw, C, tok.data_ptr(), _dev.stream())
    return _dev.to_like(tok, x)


def unpermute_euler(x, vel_curve, perm: Permutation, sigma_t: float, sigma_next: float,
                    patch=(1, 1, 1)):
    """``x + (sigma_next - sigma_t) * unpatchify(invert_permutation(vel_curve))``
    (pipeline.py:363 + 131-137) in one pass; float32 arithmetic as the reference."""
    if not sigma_next < sigma_t:
        raise DomainError(f"sigmas must decrease: {sigma_t} -> {sigma_next}")
    xt = _dev.as_cuda(x).float().contiguous()
    vt = _dev.as_cuda(vel_curve).float().contiguous()
    dims = perm.dims
    pt, ph, pw, C = _patch_dims(xt, dims, patch)
    if tuple(vt.shape) != (dims.n_cells, pt * ph * pw * C):
        raise ShapeError(f"velocity shape {tuple(vt.shape)} != {(dims.n_cells, pt * ph * pw * C)}")
    out = torch.empty_like(xt)
    _native.call("tcb_unpermute_euler", xt.data_ptr(), vt.data_ptr(), perm.inverse_dev.data_ptr(),
                 dims.t, dims.h, dims.w, pt, ph, pw, C, float(np.float32(sigma_next - sigma_t)),
                 out.data_ptr(), _dev.stream())
    return _dev.to_like(out, x)


def switch_stage_curve(x, vel_curve, perm: Permutation, sigma_t: float, target: GridDims, rng):
    """``switch_stage(x, invert_permutation(vel_curve), ...)`` with the scatter fused into
    the upsample/re-noise kernel (pipeline.py:363, 367-369)."""
    src, dst = _check_up(x, target)
    C = int(x.shape[-1])
    mode, eps, seed = _noise_source(rng, (*dst, C))  # drawn first, like pipeline.py:187
    xt = _dev.as_cuda(x).float().contiguous()
    vt = _dev.as_cuda(vel_curve).float().contiguous()
    if tuple(vt.shape) != (perm.dims.n_cells, C) or perm.dims.as_tuple() != src:
        raise ShapeError("velocity must be (n_cells, C) in the latent's curve order")
    if sigma_t in (0.0, 1.0):
        from .sfc import gather_rows

        vel = gather_rows(vt, perm.inverse_dev).reshape(xt.shape)
        x0 = predict_clean(xt, vel, sigma_t)
        if sigma_t == 0.0:
            return _dev.to_like(upsample_area_3d(x0, target), x)
        return _dev.to_like(eps if eps is not None else stage_transition(x0, 1.0, target, seed), x)
    out = torch.empty((*dst, C), dtype=torch.float32, device=xt.device)
    _native.call("tcb_upsample_renoise_curve", xt.data_ptr(), vt.data_ptr(), perm.inverse_dev.data_ptr(),
                 _native.ptr(eps), out.data_ptr(), *src, *dst, C, float(sigma_t), mode, seed, 0,
                 _dev.stream())
    return _dev.to_like(out, x)


_tables: dict = {}


def rope_tables(dims: GridDims, sections=(16, 56, 56), theta: float = 256.0,
                device=None) -> torch.Tensor:
    """(cos, sin) float32 pairs: [t x d_t/2][h x d_h/2][w x d_w/2] (float64 on the host)."""
    key = (dims.as_tuple(), tuple(sections), float(theta), str(device))
    tab = _tables.get(key)
    if tab is not None:
        return tab
    rows = []
    for n_pos, da in zip(dims.as_tuple(), sections):
        if da % 2:
            raise DomainError(f"rope sections must be even, got {sections}")
        if da == 0:
            continue
        inv_freq = theta ** (-(np.arange(0, da, 2, dtype=np.float64)) / da)
        ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv_freq[None, :]
        rows.append(np.stack([np.cos(ang), np.sin(ang)], axis=-1).reshape(-1, 2))
    host = np.concatenate(rows, axis=0).astype(np.float32) if rows else np.zeros((0, 2), np.float32)
    tab = torch.from_numpy(host).to(device or _dev.device())
    _tables[key] = tab
    return tab


def rope_permute(srcs, perm: Permutation, dsts, rotate, sections=(16, 56, 56),
                 theta: float = 256.0) -> None:
    """dst[k][hh, i, :] = rope_k(src[k][fwd[i], hh, :]) for up to 3 tensors at once.

    srcs: raster-order (n, H, d) bf16 views sharing strides (d contiguous); dsts: head-major
    (H, >= n, d) bf16 views sharing strides; rotate: per tensor, rotary embedding or copy."""
    dims = perm.dims
    n = dims.n_cells
    if not (1 <= len(srcs) == len(dsts) == len(rotate) <= 3):
        raise ShapeError("1..3 source/destination tensors")
    s0, d0 = srcs[0], dsts[0]
    if s0.ndim != 3 or s0.shape[0] != n:
        raise ShapeError(f"sources must be (n={n}, H, d), got {tuple(s0.shape)}")
    H, d = int(s0.shape[1]), int(s0.shape[2])
    for s, o in zip(srcs, dsts):
        if s.dtype != torch.bfloat16 or o.dtype != torch.bfloat16:
            raise ShapeError("rope_permute works on bfloat16 tensors")
        if s.shape != s0.shape or s.stride() != s0.stride() or s.stride(2) != 1:
            raise ShapeError("sources must share shape and strides with a contiguous last axis")
        if o.ndim != 3 or o.shape[0] != H or o.shape[1] < n or o.shape[2] != d or \
                o.stride() != d0.stride() or o.stride(2) != 1:
            raise ShapeError("destinations must be (H, >= n, d) sharing strides")
    if any(rotate) and sum(sections) != d:
        raise DomainError(f"rope sections {sections} must sum to d={d}")
    tab = rope_tables(dims, sections, theta, s0.device) if any(rotate) else None
    src_arr = (C.c_void_p * len(srcs))(*[s.data_ptr() for s in srcs])
    dst_arr = (C.c_void_p * len(dsts))(*[o.data_ptr() for o in dsts])
    rot_arr = (C.c_int * len(rotate))(*[1 if r else 0 for r in rotate])
    _native.call("tcb_rope_permute", C.cast(src_arr, C.c_void_p), s0.stride(0), s0.stride(1),
                 C.cast(dst_arr, C.c_void_p), d0.stride(0), d0.stride(1),
                 C.cast(rot_arr, C.c_void_p), len(srcs), perm.forward_dev.data_ptr(), dims.t, dims.h,
                 dims.w, H, d, _native.ptr(tab), *(sections if any(rotate) else (0, 0, 0)),
                 _dev.stream())


def qkv_to_curve(q, k, v, perm: Permutation, layout: BlockLayout, sections=(16, 56, 56),
                 theta: float = 256.0, cond=None):
    """Raster-order token-major (n, H, d) bf16 Q/K/V -> the (H, N_pad, d) curve-order buffers
    ``carve_attention`` takes, RoPE applied to Q and K, padding rows zero and the
    condition tokens (optional (q, k, v) triple of (H, n_cond, d)) copied to their rows."""
    n = perm.dims.n_cells
    if layout.n_valid != n:
        raise ShapeError(f"layout has {layout.n_valid} vision tokens, grid has {n}")
    H, d = int(q.shape[1]), int(q.shape[2])
    outs = [torch.zeros((H, layout.padded_total, d), dtype=torch.bfloat16, device=q.device)
            for _ in range(3)]
    rope_permute([q, k, v], perm, outs, [True, True, False], sections, theta)
    if cond is not None:
        for o, c in zip(outs, cond):
            if tuple(c.shape) != (H, layout.n_cond, d):
                raise ShapeError(f"condition tokens must be (H, {layout.n_cond}, {d})")
            o[:, layout.cond_start: layout.cond_start + layout.n_cond] = c
    return tuple(outs)

"""Block-sparse attention over the carve mask (reference: tokencarve attention.py).

``carve_attention`` is one carve launch: bf16 / fp16 inputs with m=128 and d in {64, 128}
run the persistent tcgen05/TMEM/TMA kernel (``tcb_carve_fwd``); fp32 inputs (the
reference's own dtype) with those shapes run the tensor-core split-fp16 kernel
(``tcb_carve_fwd_f32``, within 1e-5 of the reference); other shapes run the fp32 SIMT
kernels that mirror the reference's per-block streaming order (attention.py:162-206).  The
output has the input dtype; numpy inputs come back as float32 numpy like the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _native
from .errors import DomainError, ShapeError
from .masks import BlockMask
from .partition import BlockLayout

__all__ = ["AttentionInputs", "AmplifierBias", "compute_beta", "carve_attention",
           "dense_attention", "block_mask_logit_bias"]


@dataclass(frozen=True)
class AttentionInputs:
    """Q/K/V (heads, N, d_k) plus their layout (attention.py:35-75)."""

    q: object
    k: object
    v: object
    layout: BlockLayout

    def __post_init__(self):
        shp = [tuple(x.shape) for x in (self.q, self.k, self.v)]
        if not (shp[0] == shp[1] == shp[2]) or len(shp[0]) != 3:
            raise ShapeError(f"Q/K/V must share one (heads, N, d_k) shape, got {shp[0]}/{shp[1]}/{shp[2]}")
        if shp[0][1] != self.layout.padded_total:
            raise ShapeError(f"token axis {shp[0][1]} != padded token count {self.layout.padded_total}")

    @property
    def n_heads(self) -> int:
        return int(self.q.shape[0])

    @property
    def d_k(self) -> int:
        return int(self.q.shape[2])

    @property
    def valid_len(self) -> int:
        return self.layout.valid_len

    @property
    def text_block_start(self) -> int:
        return self.layout.M_v


@dataclass(frozen=True)
class AmplifierBias:
    """Additive logit bias on vision-query x condition-key scores (attention.py:78-86)."""

    beta: float = 0.0

    def __post_init__(self):
        if not (self.beta >= 0.0 and math.isfinite(self.beta)):
            raise DomainError(f"amplifier bias must be finite and >= 0, got {self.beta}")


def compute_beta(numel_s: int, numel_S: int, rho: float) -> float:
    """``-rho * log(numel_s / numel_S)`` (attention.py:89-96)."""
    if numel_s <= 0 or numel_S <= 0:
        raise DomainError(f"token counts must be positive, got {numel_s}, {numel_S}")
    return -rho * math.log(numel_s / numel_S) + 0.0


_work: dict = {}


def carve_work_bytes(H: int, M_v: int, M_total: int, m: int, d: int) -> int:
    """Workspace bytes tcb_carve_fwd wants for a shape (scheduler counter, plus the split
    condition rows' partials when the tcgen05 kernel runs)."""
    return int(_native.query("tcb_carve_workspace_bytes", H, M_v, M_total, m, d))


def _workspace(dev: torch.device, nbytes: int = 256) -> torch.Tensor:
    """The carve kernels' workspace (work counter + condition-row partials; the launch resets
    what it needs), one per (device, stream): launches on different streams may run
    concurrently and must not share it.  Grows to ``nbytes``; pass ``(t.data_ptr(),
    t.numel())`` as (work, work_bytes)."""
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    w = _work.get(key)
    if w is None or w.numel() < nbytes:
        w = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        _work[key] = w
    return w


def carve_raw(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mask: BlockMask,
              layout: BlockLayout, beta: float = 0.0, out: torch.Tensor | None = None,
              simt: bool = False) -> torch.Tensor:
    """Device-tensor entry: q/k/v (H, N_pad, d) of one dtype on one device, innermost axis
    contiguous (any head / token strides; all three are made contiguous if they differ)."""
    if not (q.dtype == k.dtype == v.dtype):
        raise ShapeError(f"q/k/v dtypes differ: {q.dtype}, {k.dtype}, {v.dtype}")
    if not (q.shape == k.shape == v.shape) or q.ndim != 3:
        raise ShapeError(f"q/k/v must share one (heads, N, d_k) shape")
    _dev.same_device(q, k, v, mask.words, *(() if out is None else (out,)))
    if k.stride() != q.stride() or v.stride() != q.stride() or q.stride(2) != 1:
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    with _dev.on(q):
        if out is None:
            out = torch.empty_like(q)
        if out.stride() != q.stride() or out.dtype != q.dtype or out.shape != q.shape:
            raise ShapeError("output must share the inputs' shape, dtype and strides")
        launch_carve(q, k, v, out, mask.words, mask.kv_cnt, layout.m, layout.M_v, layout.M_total,
                     layout.n_valid, layout.n_cond, beta, simt)
    return out


def launch_carve(q, k, v, out, words, kv_cnt, m, M_v, M_total, n_valid, n_cond, beta,
                 simt: bool = False) -> None:
    """The carve launch shared by carve_raw and the torch op: bf16 / fp16 -> tcgen05 kernel;
    fp32 -> tensor-core split-fp16 kernel (the library itself falls back to the fp32 SIMT
    kernel for shapes that path does not take); ``simt`` forces the fp32 SIMT kernel."""
    H, N, d = q.shape
    args = (q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), _dev.code_of(q.dtype),
            q.stride(0), q.stride(1), words.data_ptr(), words.shape[-1], kv_cnt.data_ptr(), H, d,
            m, M_v, M_total, n_valid, n_cond, float(beta))
    if simt:
        _native.call("tcb_carve_fwd_simt", *args, _dev.stream())
    elif q.dtype == torch.float32:
        nb = _native.query("tcb_carve_f32_workspace_bytes", H, M_total, m, d)
        ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=q.device)
        _native.call("tcb_carve_fwd_f32", *args[:4], *args[5:], ws.data_ptr(), nb,
                     _workspace(q.device).data_ptr(), _dev.stream())
    else:
        w = _workspace(q.device, carve_work_bytes(H, M_v, M_total, m, d))
        _native.call("tcb_carve_fwd", *args, w.data_ptr(), w.numel(), _dev.stream())


def carve_attention(inputs: AttentionInputs, mask: BlockMask,
                    beta: AmplifierBias = AmplifierBias(0.0), n_workers: int | None = None):
    """Block-sparse attention (attention.py:209-243).

    ``n_workers`` is accepted for signature compatibility and ignored (results never
    depend on it; the kernel's kv visit order is fixed ascending).
    """
    layout = inputs.layout
    expected = (inputs.n_heads, layout.M_v, layout.M_total)
    if tuple(mask.shape) != expected:
        raise ShapeError(f"mask shape {tuple(mask.shape)} != {expected}")
    if layout.M_v:
        mask.check_nonempty()
    q, k, v = (_dev.as_cuda(x) for x in (inputs.q, inputs.k, inputs.v))
    _dev.same_device(q, k, v)
    if not (q.dtype == k.dtype == v.dtype) or q.dtype not in (torch.float32, torch.bfloat16,
                                                               torch.float16):
        # mixed or other dtypes compute in float32, as the reference's astype(float32)
        q, k, v = q.float(), k.float(), v.float()
    out = carve_raw(q, k, v, mask, layout, beta.beta)
    return _dev.to_like(out, inputs.q)


def _valid_keys(n: int, valid, device) -> torch.Tensor:
    if valid is None:
        return torch.ones(n, dtype=torch.bool, device=device)
    if isinstance(valid, (int, np.integer)):
        ok = torch.zeros(n, dtype=torch.bool, device=device)
        ok[: int(valid)] = True
        return ok
    ok = _dev.as_cuda(np.asarray(valid, dtype=bool) if not isinstance(valid, torch.Tensor) else valid)
    if tuple(ok.shape) != (n,):
        raise ShapeError(f"valid mask shape {tuple(ok.shape)} != ({n},)")
    return ok.to(torch.bool)


def dense_attention(q, k, v, logit_bias=None, valid=None):
    """Exact two-pass fp32 softmax attention (attention.py:112-142): the dense check the
    reference CLI runs against carve output.  fp32 GEMMs (cuBLAS, TF32 off) on the device;
    ``logit_bias`` broadcastable to (H, N, N) with -inf dropping pairs; padding keys get
    -inf and padding query rows are zeroed.  Not a hot-path kernel."""
    shp = [tuple(x.shape) for x in (q, k, v)]
    if not (shp[0] == shp[1] == shp[2]) or len(shp[0]) != 3:
        raise ShapeError(f"Q/K/V must share one (heads, N, d_k) shape, got {shp[0]}")
    H, n, d_k = shp[0]
    qd, kd, vd = (_dev.as_cuda(x).float() for x in (q, k, v))
    ok = _valid_keys(n, valid, qd.device)
    scale = np.float32(1.0 / math.sqrt(d_k))
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        scores = torch.matmul(qd * float(scale), kd.transpose(1, 2))
        if logit_bias is not None:
            scores = scores + _dev.as_cuda(logit_bias).float()
        scores = torch.where(ok[None, None, :], scores, torch.tensor(float("-inf"), device=qd.device))
        scores = scores - scores.amax(dim=-1, keepdim=True)
        w = torch.exp(scores)
        w = w / w.sum(dim=-1, keepdim=True)
        out = torch.matmul(w, vd)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    out[:, ~ok, :] = 0.0
    return _dev.to_like(out, q)


def block_mask_logit_bias(mask: BlockMask, layout: BlockLayout, beta: float = 0.0):
    """Token-level additive bias equivalent to a block mask + amplifier
    (attention.py:145-159): -inf on deselected vision-row blocks, condition rows open,
    +beta on vision-query x condition-key pairs.  Built on the device."""
    m, n = layout.m, layout.padded_total
    bits = mask.bits_dev if isinstance(mask, BlockMask) else _dev.as_cuda(mask)
    H = int(bits.shape[0])
    bias = torch.zeros((H, layout.M_total, layout.M_total), dtype=torch.float32, device=bits.device)
    bias[:, : layout.M_v, :] = torch.where(bits.to(torch.bool), 0.0, float("-inf"))
    if beta:
        bias[:, : layout.M_v, layout.M_v:] += np.float32(beta)
    out = bias.repeat_interleave(m, dim=1).repeat_interleave(m, dim=2).reshape(H, n, n)
    host = mask.host if isinstance(mask, BlockMask) else isinstance(mask, np.ndarray)
    return out.cpu().numpy() if host else out

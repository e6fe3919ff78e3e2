"""Progressive-resolution sampler around the carved-attention path, on the device
(reference: tokencarve pipeline.py).

Hot pieces run as kernels: the stage switch ``predict_clean -> upsample ->
re-noise`` is one launch of ``tcb_upsample_renoise`` (K9/K10), the per-step
curve permute/unpermute is the K2 gather, the per-stage curve and adjacency are
K1/K6.  Schedules, plans and the loop itself are host bookkeeping
(O(steps) scalars) restated from pipeline.py:49-121, 224-391.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _dev, _native
from .attention import AmplifierBias, AttentionInputs, carve_attention, compute_beta
from .errors import ContractError, DomainError, ShapeError
from .masks import SelectionParams, build_block_mask
from .partition import BlockLayout, StaticMasks, build_layout
from .sfc import GridDims, Permutation, build_curve, gather_rows

__all__ = ["SigmaSchedule", "StageConfig", "StagePlan", "StepContext", "PipelineResult",
           "shifted_sigmas", "skip_schedule", "predict_clean", "denoise_step", "upsample_area_3d",
           "stage_transition", "switch_stage", "toy_transformer_denoiser", "run_pipeline",
           "plan_from_dict", "plan_to_dict"]


# ----------------------------------------------------------------------------- schedules
@dataclass(frozen=True)
class SigmaSchedule:
    """Strictly decreasing sigmas ending at 0 (pipeline.py:49-69)."""

    sigmas: np.ndarray

    def __post_init__(self):
        s = self.sigmas
        if s.ndim != 1 or s.shape[0] < 2:
            raise ShapeError("sigma schedule needs at least one step plus the terminal 0")
        if s[-1] != 0.0:
            raise DomainError("sigma schedule must end at exactly 0")
        if not np.all(np.diff(s) < 0):
            raise DomainError("sigmas must be strictly decreasing")
        if s[0] > 1.0 or s[-2] <= 0.0:
            raise DomainError("retained sigmas must lie in (0, 1]")
        s.setflags(write=False)

    @property
    def n_steps(self) -> int:
        return self.sigmas.shape[0] - 1


def shifted_sigmas(step_indices, base_T: int, alpha: float) -> SigmaSchedule:
    """sigma = alpha*u / (1 + (alpha-1)*u), u = (T - j)/T (pipeline.py:72-92)."""
    if alpha < 1.0:
        raise DomainError(f"shift factor must be >= 1, got {alpha}")
    idx = np.asarray(step_indices, dtype=np.int64)
    if idx.ndim != 1 or idx.size == 0:
        raise ShapeError("step_indices must be a non-empty 1D sequence")
    if idx.min() < 0 or idx.max() >= base_T:
        raise DomainError(f"step indices must lie in [0, {base_T})")
    if np.any(np.diff(idx) <= 0):
        raise DomainError("step indices must be strictly ascending")
    u = (base_T - idx.astype(np.float64)) / base_T
    return SigmaSchedule(sigmas=np.concatenate([alpha * u / (1.0 + (alpha - 1.0) * u), [0.0]]))


def skip_schedule(base_T: int, keep: int) -> list:
    """Dense-ends retained steps by highest-averages gap allocation (pipeline.py:95-121)."""
    if not (1 <= keep <= base_T):
        raise DomainError(f"keep must be in [1, {base_T}], got {keep}")
    if keep == base_T:
        return list(range(base_T))
    if keep == 1:
        return [0]
    n = keep - 1
    extra = (base_T - 1) - n
    x = (np.arange(n) - (n - 1) / 2.0) / max(n - 1, 1) * 2.0
    weight = 1.0 + 4.0 * (1.0 - x ** 2)
    alloc = np.zeros(n, dtype=np.int64)
    dist = np.abs(x)
    for _ in range(extra):
        quotient = weight / (alloc + 1)
        alloc[np.lexsort((np.arange(n), dist, -quotient))[0]] += 1
    return [0] + np.cumsum(1 + alloc).tolist()


@dataclass(frozen=True)
class StageConfig:
    dims: GridDims
    step_indices: tuple
    alpha: float
    k: float = 0.3
    rho: float = 0.0


@dataclass(frozen=True)
class StagePlan:
    """Stages + shared sampling knobs (pipeline.py:233-269)."""

    stages: tuple
    base_T: int = 50
    block_size: int = 128
    n_cond_tokens: int = 0
    p: float = 0.3

    def __post_init__(self):
        if not self.stages:
            raise ContractError("a plan needs at least one stage")
        prev = None
        for i, st in enumerate(self.stages):
            idx = np.asarray(st.step_indices)
            if idx.size == 0 or idx.min() < 0 or idx.max() >= self.base_T:
                raise DomainError(f"stage {i}: step indices must lie in [0, {self.base_T})")
            if st.alpha < 1.0:
                raise DomainError(f"stage {i}: shift factor must be >= 1")
            if i > 0 and st.rho != 0.0:
                raise ContractError("the text amplifier resets after stage 1 (rho = 0)")
            if prev is not None and any(d < p for p, d in zip(prev.as_tuple(), st.dims.as_tuple())):
                raise ContractError("stage resolutions must be nondecreasing per axis")
            prev = st.dims

    @property
    def target_dims(self) -> GridDims:
        return self.stages[-1].dims

    @property
    def n_evaluations(self) -> int:
        return sum(len(s.step_indices) for s in self.stages)


def plan_from_dict(data: dict) -> StagePlan:
    try:
        stages = tuple(StageConfig(dims=GridDims(*s["dims"]), step_indices=tuple(int(i) for i in s["steps"]),
                                   alpha=float(s["alpha"]), k=float(s.get("k", 0.3)),
                                   rho=float(s.get("rho", 0.0))) for s in data["stages"])
    except (KeyError, TypeError) as exc:
        raise ContractError(f"malformed plan: {exc}") from exc
    return StagePlan(stages=stages, base_T=int(data.get("base_steps", 50)),
                     block_size=int(data.get("block_size", 128)),
                     n_cond_tokens=int(data.get("cond_tokens", 0)), p=float(data.get("p", 0.3)))


def plan_to_dict(plan: StagePlan) -> dict:
    return {"stages": [{"dims": list(s.dims.as_tuple()), "steps": list(s.step_indices),
                        "alpha": s.alpha, "k": s.k, "rho": s.rho} for s in plan.stages],
            "base_steps": plan.base_T, "block_size": plan.block_size,
            "cond_tokens": plan.n_cond_tokens, "p": plan.p}


# ----------------------------------------------------------------------------- point ops
def _pair(a, b):
    """Device views of two same-shape latents in their common float dtype (float32, or
    float64 when either is float64 -- numpy's promotion for the reference's expressions)."""
    x, y = _dev.as_cuda(a), _dev.as_cuda(b)
    dt = torch.float64 if torch.float64 in (x.dtype, y.dtype) else torch.float32
    return x.to(dt).contiguous(), y.to(dt).contiguous()


def _axpy(x: torch.Tensor, y: torch.Tensor, coef: float) -> torch.Tensor:
    """``x + coef * y`` elementwise in x's dtype (coef rounded to it, like
    np.asarray(coef, dtype=x.dtype)), one K9 Euler launch."""
    _dev.same_device(x, y)
    with _dev.on(x):
        out = torch.empty_like(x)
        if x.dtype == torch.float64:
            _native.call("tcb_euler_step_f64", x.data_ptr(), y.data_ptr(), out.data_ptr(),
                         x.numel(), float(coef), _dev.stream())
        else:
            _native.call("tcb_euler_step", x.data_ptr(), y.data_ptr(), out.data_ptr(), x.numel(),
                         float(np.float32(coef)), _dev.stream())
    return out


def _f32(x) -> torch.Tensor:
    t = _dev.as_cuda(x)
    if t.dtype != torch.float32:
        raise TypeError("latents are float32")
    return t.contiguous()


def predict_clean(x_t, eps_t, sigma_t: float):
    """``x - sigma * eps`` (pipeline.py:124-128), float32 or float64 like the input."""
    if tuple(x_t.shape) != tuple(eps_t.shape):
        raise ShapeError(f"latent and prediction shapes differ: {tuple(x_t.shape)} vs {tuple(eps_t.shape)}")
    x, e = _pair(x_t, eps_t)
    # x + (-sigma) * e == x - sigma * e bitwise in IEEE arithmetic
    return _dev.to_like(_axpy(x, e, -sigma_t), x_t)


def denoise_step(x_t, v_t, sigma_t: float, sigma_next: float):
    """Euler step ``x + (sigma_next - sigma) * v`` (pipeline.py:131-137)."""
    if tuple(x_t.shape) != tuple(v_t.shape):
        raise ShapeError(f"latent and velocity shapes differ: {tuple(x_t.shape)} vs {tuple(v_t.shape)}")
    if not sigma_next < sigma_t:
        raise DomainError(f"sigmas must decrease: {sigma_t} -> {sigma_next}")
    x, v = _pair(x_t, v_t)
    return _dev.to_like(_axpy(x, v, sigma_next - sigma_t), x_t)


def _check_up(x, target: GridDims):
    if x.ndim != 4:
        raise ShapeError(f"latent must be rank 4 (t, h, w, c), got shape {tuple(x.shape)}")
    src, dst = tuple(int(v) for v in x.shape[:3]), target.as_tuple()
    if any(d < s for s, d in zip(src, dst)):
        raise DomainError(f"target {dst} shrinks source {src}")
    return src, dst


def _latent(x) -> torch.Tensor:
    """Device latent in float32, or float64 kept as is (the reference upsamples in float64)."""
    t = _dev.as_cuda(x)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float32)
    return t.contiguous()


def _launch_switch(x: torch.Tensor, vel, eps, sigma: float, dst, mode: int, seed: int = 0,
                   offset: int = 0) -> torch.Tensor:
    C = x.shape[-1]
    with _dev.on(x):
        if x.dtype == torch.float64:
            odt = torch.float64 if mode == 0 else torch.float32
            out = torch.empty((*dst, C), dtype=odt, device=x.device)
            _native.call("tcb_upsample_renoise_f64", x.data_ptr(), _native.ptr(eps), out.data_ptr(),
                         *x.shape[:3], *dst, C, float(sigma), mode, seed, offset, _dev.stream())
            return out
        out = torch.empty((*dst, C), dtype=torch.float32, device=x.device)
        _native.call("tcb_upsample_renoise", x.data_ptr(), _native.ptr(vel), _native.ptr(eps),
                     out.data_ptr(), *x.shape[:3], *dst, C, float(sigma), mode, seed, offset,
                     _dev.stream())
    return out


def upsample_area_3d(x, target: GridDims):
    """Area upsample of a (t, h, w, c) latent (pipeline.py:153-173); float64 input stays
    float64, like the reference's ``astype(x.dtype)``."""
    src, dst = _check_up(x, target)
    xt = _latent(x)
    if src == dst:
        return x.copy() if _dev.is_numpy(x) else xt.clone()
    return _dev.to_like(_launch_switch(xt, None, None, 0.0, dst, 0), x)


def _noise_source(rng, shape):
    """numpy Generator -> host-drawn eps (bitwise reference parity, mode 1);
    torch.Generator / int seed -> in-kernel Philox (mode 2)."""
    if isinstance(rng, np.random.Generator):
        eps = rng.standard_normal(shape, dtype=np.float32)
        return 1, _dev.as_cuda(eps), 0
    if isinstance(rng, torch.Generator):
        seed = int(torch.randint(0, 2**62, (1,), generator=rng).item())
    else:
        seed = int(rng)
    return 2, None, seed


def stage_transition(x0, sigma_t: float, target: GridDims, rng):
    """``(1 - s) * upsample(x0) + s * eps`` (pipeline.py:176-194)."""
    if not (0.0 <= sigma_t <= 1.0):
        raise DomainError(f"transition sigma must be in [0, 1], got {sigma_t}")
    src, dst = _check_up(x0, target)
    C = int(x0.shape[-1])
    mode, eps, seed = _noise_source(rng, (*dst, C))  # drawn first, like pipeline.py:187
    xt = _latent(x0)
    if sigma_t == 0.0:
        return upsample_area_3d(x0, target)
    if sigma_t == 1.0:
        if eps is None:
            eps = _launch_switch(torch.zeros((*dst, C), device=xt.device), None, None, 1.0, dst,
                                 2, seed)
        return _dev.to_like(eps, x0)
    return _dev.to_like(_launch_switch(xt, None, eps, sigma_t, dst, mode, seed), x0)


def switch_stage(x, vel, sigma_t: float, target: GridDims, rng):
    """Fused ``stage_transition(predict_clean(x, vel, sigma), sigma, target, rng)``:
    one K9/K10 launch (pipeline.py:367-369)."""
    src, dst = _check_up(x, target)
    C = int(x.shape[-1])
    mode, eps, seed = _noise_source(rng, (*dst, C))
    xt, vt = _f32(x), _f32(vel)
    if sigma_t in (0.0, 1.0):
        x0 = predict_clean(xt, vt, sigma_t)
        if sigma_t == 0.0:
            return _dev.to_like(upsample_area_3d(x0, target), x)
        return _dev.to_like(eps if eps is not None else stage_transition(x0, 1.0, target, seed), x)
    return _dev.to_like(_launch_switch(xt, vt, eps, sigma_t, dst, mode, seed), x)


# ----------------------------------------------------------------------------- analytic denoiser
def gaussian_posterior_mean(x_t, sigma: float, mu: float, s: float):
    """E[x0 | x_t] for x0 ~ N(mu, s^2 I), x_t = (1-sigma) x0 + sigma eps
    (pipeline.py:195-199); same scalar/array operation order as the reference."""
    a = 1.0 - sigma
    denom = a * a * s * s + sigma * sigma
    return mu + a * s * s * (x_t - a * mu) / denom


def gaussian_analytic_denoiser(mu: float, s: float) -> "Denoiser":
    """Exact velocity E[eps - x0 | x_t] for Gaussian data (pipeline.py:202-221), as an
    elementwise expression on the device tokens (float32 result like the input)."""
    if s <= 0:
        raise DomainError(f"data std must be positive, got {s}")
    s2 = s * s

    def velocity(tokens, ctx: "StepContext"):
        tok = _dev.as_cuda(tokens)
        sig = ctx.sigma
        a = 1.0 - sig
        denom = a * a * s2 + sig * sig
        # numpy >= 2 keeps Python scalars weak: every op runs in the array's dtype (float32
        # for latents) with the scalar rounded to it, as torch does; the divisor is a 0-dim
        # tensor so the division is a true per-element divide (a CPU-scalar divide would
        # multiply by 1/denom).  numpy callers get numpy back.
        t = tok if tok.dtype == torch.float64 else tok.float()
        num = sig * (t - mu) - a * s2 * t
        return _dev.to_like(num / torch.tensor(denom, dtype=t.dtype, device=t.device), tokens)

    return velocity


# ----------------------------------------------------------------------------- loop
@dataclass
class StepContext:
    """Per-evaluation context handed to the denoiser (pipeline.py:272-292)."""

    stage: int
    step_index: int
    sigma: float
    dims: GridDims
    layout: BlockLayout
    perm: Permutation
    statics: StaticMasks
    positions: torch.Tensor
    params: SelectionParams
    beta: AmplifierBias
    metrics: dict = field(default_factory=dict)


Denoiser = Callable[[torch.Tensor, StepContext], torch.Tensor]


@dataclass
class PipelineResult:
    latent: object
    report: dict


def run_pipeline(plan: StagePlan, denoiser: Denoiser, rng=0, channels: int = 1) -> PipelineResult:
    """All stages of the plan on the device (pipeline.py:304-391).

    ``rng`` is a numpy Generator / seed (noise drawn on the host like the reference,
    so runs are comparable bitwise in their noise) -- tokens, velocities and the
    latent stay on the device; the terminal latent is returned as numpy.
    """
    from .fused import curve_positions, switch_stage_curve, unpermute_euler

    if not isinstance(rng, np.random.Generator):
        rng = np.random.default_rng(rng)
    t0 = time.perf_counter()
    target_numel = plan.target_dims.n_cells
    x = _dev.as_cuda(rng.standard_normal((*plan.stages[0].dims.as_tuple(), channels),
                                         dtype=np.float32))
    stage_reports, step_records = [], []
    for s_idx, stage in enumerate(plan.stages):
        dims = stage.dims
        n = dims.n_cells
        perm = build_curve(dims)
        layout = build_layout(dims, plan.block_size, plan.n_cond_tokens)
        statics = StaticMasks.build(layout, dims, perm)
        positions = curve_positions(perm)  # one pass from fwd (pipeline.py:334-337)
        beta = AmplifierBias(compute_beta(n, target_numel, stage.rho))
        params = SelectionParams(k=stage.k, p=plan.p)
        schedule = shifted_sigmas(stage.step_indices, plan.base_T, stage.alpha)
        last = len(stage.step_indices) - 1
        for j, idx in enumerate(stage.step_indices):
            sigma = float(schedule.sigmas[j])
            z = gather_rows(x.reshape(n, channels), perm.forward_dev)
            ctx = StepContext(stage=s_idx, step_index=int(idx), sigma=sigma, dims=dims,
                              layout=layout, perm=perm, statics=statics, positions=positions,
                              params=params, beta=beta)
            vel_curve = _dev.as_cuda(denoiser(z, ctx))
            if tuple(vel_curve.shape) != tuple(z.shape):
                raise ShapeError(f"denoiser returned shape {tuple(vel_curve.shape)}, expected {tuple(z.shape)}")
            step_records.append({"stage": s_idx, "step_index": int(idx), "sigma": sigma,
                                 **ctx.metrics})
            # invert_permutation fused into the update / switch (pipeline.py:363-371)
            if s_idx < len(plan.stages) - 1 and j == last:
                x = switch_stage_curve(x, vel_curve, perm, sigma, plan.stages[s_idx + 1].dims, rng)
            else:
                x = unpermute_euler(x, vel_curve, perm, sigma, float(schedule.sigmas[j + 1]))
        stage_reports.append({"stage": s_idx, "dims": list(dims.as_tuple()), "n_tokens": n,
                              "token_ratio_to_target": n / target_numel,
                              "n_steps": len(stage.step_indices), "alpha": stage.alpha,
                              "beta": beta.beta})
    report = {"stages": stage_reports, "steps": step_records,
              "n_evaluations": plan.n_evaluations, "wall_time": time.perf_counter() - t0}
    return PipelineResult(latent=x.cpu().numpy(), report=report)


def toy_transformer_denoiser(channels: int = 1, n_heads: int = 2, d_k: int = 16,
                             seed: int = 1234) -> Denoiser:
    """Fixed random-weight attention denoiser (pipeline.py:394-439) on the device:
    projections are plain fp32 matmuls, the attention stack is the carve path."""
    g = np.random.default_rng(seed)
    f_in = channels + 3
    sc = 1.0 / math.sqrt(f_in)
    w_q = (g.standard_normal((n_heads, f_in, d_k)) * sc).astype(np.float32)
    w_k = (g.standard_normal((n_heads, f_in, d_k)) * sc).astype(np.float32)
    w_v = (g.standard_normal((n_heads, f_in, d_k)) * sc).astype(np.float32)
    w_o = (g.standard_normal((n_heads * d_k, channels)) / math.sqrt(n_heads * d_k)).astype(np.float32)
    W = {}

    def weights(dev):
        if dev not in W:
            W[dev] = tuple(torch.from_numpy(a).to(dev) for a in (w_q, w_k, w_v, w_o))
        return W[dev]

    def velocity(tokens, ctx: StepContext):
        layout = ctx.layout
        tok = _dev.as_cuda(tokens).float()
        wq, wk, wv, wo = weights(tok.device)
        dims = torch.tensor(ctx.dims.as_tuple(), dtype=torch.float32, device=tok.device)
        pos = ctx.positions.float() / torch.clamp(dims, min=1.0)
        feats = torch.cat([tok, pos], dim=1)
        padded = torch.zeros((layout.padded_total, f_in), dtype=torch.float32, device=tok.device)
        padded[: layout.n_valid] = feats
        if layout.n_cond:
            cg = np.random.default_rng(seed + 1)
            padded[layout.cond_start: layout.cond_start + layout.n_cond] = torch.from_numpy(
                cg.standard_normal((layout.n_cond, f_in)).astype(np.float32)).to(tok.device)
        q = torch.einsum("nf,hfd->hnd", padded, wq).contiguous()
        k = torch.einsum("nf,hfd->hnd", padded, wk).contiguous()
        v = torch.einsum("nf,hfd->hnd", padded, wv).contiguous()
        mask, _ = build_block_mask(q, k, layout, ctx.statics, ctx.params, need_relevance=False)
        out = carve_attention(AttentionInputs(q=q, k=k, v=v, layout=layout), mask, ctx.beta)
        ctx.metrics["effective_sparsity"] = 1.0 - mask.selected_fraction
        merged = out.permute(1, 0, 2).reshape(layout.padded_total, n_heads * d_k)
        return merged[: layout.n_valid] @ wo - tok

    return velocity

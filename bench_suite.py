"""Secondary measurements for SURVEY.md §8 configs beyond the bench.py headline (C2):

  * hbm kernels at C2: permute (118,800 x 3,072 bf16 gather), block pool (Q+K), curve
    build, adjacency build -- achieved GB/s vs the measured HBM peak;
  * C3: Wan2.1-14B 480p layer (21x30x52, H=40, no text), k=0.08 -- ms/layer, TFLOP/s;
  * C4: ProRes 2-stage switch at 720p: fused predict_clean+upsample+renoise
    (33,34,60,16) -> (33,45,80,16), curve + adjacency rebuild at the new dims, and
    one toy-width permute of the latent;
  * C5: sparsity sweep on C2, k in {0.01, 0.02, 0.05, 0.08, 0.10, 0.20, 0.30}, p=0;
  * §8f-1 fused neighbours at C2: QKV -> curve-order head-major with 3D RoPE (vs the
    unfused torch composition), unpermute+Euler, curve positions.

All timings: CUDA events on the launching stream, median of repeats after warm-up.
Writes one JSON document (stdout, and --out if given).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import paper_2505_16864_b200 as tcb  # noqa: E402
from paper_2505_16864_b200 import _native  # noqa: E402
from paper_2505_16864_b200.attention import _workspace, carve_work_bytes  # noqa: E402
from paper_2505_16864_b200.masks import mask_scratch, launch_mask, mask_buffers  # noqa: E402
from paper_2505_16864_b200.partition import mask_words  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return p["hbm_gbs"], p["bf16_tflops"]
    except Exception:
        return 6650.0, 1590.0


class Layer:
    """Device buffers + the launches of one carved-attention layer."""

    def __init__(self, dims, n_cond, H, k_rate, seed=0, p_cut=0.0, beta=0.0):
        self.dims = tcb.GridDims(*dims)
        self.lay = tcb.build_layout(self.dims, 128, n_cond)
        self.st = tcb.StaticMasks.build(self.lay, self.dims, tcb.build_curve(self.dims))
        self.adja = self.st.packed(self.lay)
        self.H, self.k, self.p, self.beta = H, k_rate, p_cut, beta
        L = self.lay
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)
        self.q, self.kk, self.v = (torch.randn((H, L.padded_total, 128), generator=g, device="cuda")
                                   .to(torch.bfloat16) for _ in range(3))
        self.o = torch.empty_like(self.q)
        self.pq = torch.empty((H, L.M_total, 128), dtype=torch.float64, device="cuda")
        self.pk = torch.empty_like(self.pq)
        self.words = mask_words(L.M_total)
        self.bits, self.kv_cnt = mask_buffers(H, L, self.q.device)
        self.scratch = mask_scratch(H, L, self.q.device)
        self.work = _workspace(self.q.device, carve_work_bytes(H, L.M_v, L.M_total, 128, 128))
        self.s = torch.cuda.current_stream().cuda_stream

    def mask(self):
        L, H = self.lay, self.H
        _native.call("tcb_block_pool", self.q.data_ptr(), self.kk.data_ptr(), 1, self.q.stride(0),
                     self.q.stride(1), H, 128, 128, L.M_v, L.M_total, L.n_valid, L.n_cond,
                     self.pq.data_ptr(), self.pk.data_ptr(), self.s)
        launch_mask(self.pq, self.pk, L, self.adja, tcb.SelectionParams(k=self.k, p=self.p),
                    self.bits, self.kv_cnt, self.s, self.scratch)

    def carve(self):
        L = self.lay
        _native.call("tcb_carve_fwd", self.q.data_ptr(), self.kk.data_ptr(), self.v.data_ptr(),
                     self.o.data_ptr(), 1, self.q.stride(0), self.q.stride(1),
                     self.bits.data_ptr(), self.words, self.kv_cnt.data_ptr(), self.H, 128, 128, L.M_v,
                     L.M_total, L.n_valid, L.n_cond, float(self.beta), self.work.data_ptr(),
                     self.work.numel(), self.s)

    def pairs(self):
        return int(self.kv_cnt.sum().item()) + self.H * self.lay.M_c * self.lay.M_total


def layer_record(name, dims, n_cond, H, k, p=0.0, beta=0.0):
    lay = Layer(dims, n_cond, H, k, p_cut=p, beta=beta)
    t_mask = timed(lay.mask)
    lay.mask()
    t_carve = timed(lay.carve)
    pairs = lay.pairs()
    flops = 4.0 * 128 * 128 * 128 * pairs
    _, tf = peaks()
    rec = {"config": name, "dims": list(dims), "heads": H, "k": k, "p": p, "beta": beta,
           "kept_pairs": pairs, "kept_fraction": round(pairs / (H * lay.lay.M_total ** 2), 4),
           "mask_ms": round(t_mask, 4), "carve_ms": round(t_carve, 4),
           "layer_ms": round(t_mask + t_carve, 4),
           "kept_tflops": round(flops / (t_carve * 1e-3) / 1e12, 1),
           "frac_of_measured_bf16": round(flops / (t_carve * 1e-3) / 1e12 / tf, 4)}
    del lay
    torch.cuda.empty_cache()
    return rec


def hbm_records():
    hbm, _ = peaks()
    out = []
    dims = tcb.GridDims(33, 45, 80)
    perm = tcb.build_curve(dims)
    n = dims.n_cells
    x = torch.randn((n, 3072), device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    t = timed(lambda: tcb.gather_rows(x, perm.forward_dev, out=y), reps=20)
    byts = 2 * x.numel() * 2 + 4 * n
    out.append({"kernel": "permute_rows (K2)", "shape": "118800 x 3072 bf16", "ms": round(t, 4),
                "gbs": round(byts / (t * 1e-3) / 1e9, 1), "frac_of_hbm": round(byts / (t * 1e-3) / 1e9 / hbm, 3)})
    del x, y
    lay = tcb.build_layout(dims, 128, 256)
    q = torch.randn((24, lay.padded_total, 128), device="cuda").to(torch.bfloat16)
    k = torch.randn_like(q)
    pq = torch.empty((24, lay.M_total, 128), dtype=torch.float64, device="cuda")
    pk = torch.empty_like(pq)
    s = torch.cuda.current_stream().cuda_stream
    t = timed(lambda: _native.call("tcb_block_pool", q.data_ptr(), k.data_ptr(), 1, q.stride(0), q.stride(1), 24,
                                   128, 128, lay.M_v, lay.M_total, lay.n_valid, lay.n_cond, pq.data_ptr(),
                                   pk.data_ptr(), s), reps=20)
    byts = 2 * q.numel() * 2 + 2 * pq.numel() * 8
    out.append({"kernel": "block_pool Q+K (K3)", "shape": "2 x 24 x 119168 x 128 bf16", "ms": round(t, 4),
                "gbs": round(byts / (t * 1e-3) / 1e9, 1), "frac_of_hbm": round(byts / (t * 1e-3) / 1e9 / hbm, 3)})
    del q, k
    fwd = torch.empty(n, dtype=torch.int32, device="cuda")
    inv = torch.empty_like(fwd)
    t = timed(lambda: _native.call("tcb_curve_build", 33, 45, 80, fwd.data_ptr(), inv.data_ptr(), s), reps=20)
    out.append({"kernel": "curve_build (K1)", "shape": "33x45x80", "ms": round(t, 4),
                "gbs": round(8 * n / (t * 1e-3) / 1e9, 1), "note": "latency bound (0.95 MB written)"})
    words = mask_words(lay.M_total)
    adja = torch.empty((lay.M_v, words), dtype=torch.int32, device="cuda")
    t = timed(lambda: _native.call("tcb_adjacency_build", inv.data_ptr(), 33, 45, 80, 128, lay.M_v, words,
                                   adja.data_ptr(), s), reps=20)
    out.append({"kernel": "adjacency_build (K6)", "shape": "33x45x80, m=128", "ms": round(t, 4),
                "note": "13 neighbour offsets per cell, packed atomics"})
    return out


def c4_records():
    hbm, _ = peaks()
    src, dst, C = (33, 34, 60), tcb.GridDims(33, 45, 80), 16
    x = torch.randn((*src, C), device="cuda")
    vel = torch.randn_like(x)
    eps = torch.randn((*dst.as_tuple(), C), device="cuda")
    out = torch.empty_like(eps)
    s = torch.cuda.current_stream().cuda_stream
    t = timed(lambda: _native.call("tcb_upsample_renoise", x.data_ptr(), vel.data_ptr(), eps.data_ptr(),
                                   out.data_ptr(), *src, *dst.as_tuple(), C, 0.899083, 1, 0, 0, s), reps=20)
    byts = 2 * x.numel() * 4 + 2 * out.numel() * 4
    recs = [{"kernel": "upsample_renoise (K9/K10, eps supplied)", "shape": "(33,34,60,16)->(33,45,80,16)",
             "ms": round(t, 4), "gbs": round(byts / (t * 1e-3) / 1e9, 1)}]
    t = timed(lambda: _native.call("tcb_upsample_renoise", x.data_ptr(), vel.data_ptr(), None, out.data_ptr(),
                                   *src, *dst.as_tuple(), C, 0.899083, 2, 1234, 0, s), reps=20)
    recs.append({"kernel": "upsample_renoise (K9/K10, in-kernel Philox)", "shape": "(33,34,60,16)->(33,45,80,16)",
                 "ms": round(t, 4), "gbs": round((byts - out.numel() * 4) / (t * 1e-3) / 1e9, 1)})

    def switch():
        perm = tcb.build_curve(dst)
        lay = tcb.build_layout(dst, 128, 256)
        tcb.StaticMasks.build(lay, dst, perm)
        z = tcb.switch_stage(x, vel, 0.899083, dst, 1234)
        tcb.gather_rows(z.reshape(-1, C), perm.forward_dev)

    t = timed(switch, reps=10)
    recs.append({"kernel": "full stage switch (switch + curve + statics + permute)", "ms": round(t, 4),
                 "note": "includes host-side launches of 6 kernels"})
    return recs


def fused_records():
    """§8f-1 fused neighbours at C2: QKV raster -> curve head-major with 3D RoPE (one pass)
    vs the unfused torch composition (gather, rotate, transpose), plus the per-step
    latent kernels."""
    from paper_2505_16864_b200 import fused

    hbm, _ = peaks()
    dims = tcb.GridDims(33, 45, 80)
    perm = tcb.build_curve(dims)
    lay = tcb.build_layout(dims, 128, 256)
    n, H, d = dims.n_cells, 24, 128
    qkv = torch.randn((n, 3, H, d), device="cuda").to(torch.bfloat16)
    outs = [torch.zeros((H, lay.padded_total, d), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    srcs = [qkv[:, 0], qkv[:, 1], qkv[:, 2]]
    fused.rope_tables(dims)
    t = timed(lambda: fused.rope_permute(srcs, perm, outs, [True, True, False]), reps=20)
    byts = 2 * 3 * n * H * d * 2 + 4 * n
    recs = [{"kernel": "rope_permute Q/K/V (3D RoPE on Q,K; raster token-major -> curve head-major)",
             "shape": "118800 x 3 x 24 x 128 bf16", "ms": round(t, 4),
             "gbs": round(byts / (t * 1e-3) / 1e9, 1), "frac_of_hbm": round(byts / (t * 1e-3) / 1e9 / hbm, 3)}]
    # unfused torch composition of the same result (for the traffic comparison)
    tab = fused.rope_tables(dims).view(-1, 2)
    pos = fused.curve_positions(perm)
    sec = (16, 56, 56)
    offs = [0, dims.t * 8, dims.t * 8 + dims.h * 28]
    cs = torch.cat([tab[offs[a] + pos[:, a:a + 1] * (sec[a] // 2) +
                        torch.arange(sec[a] // 2, device="cuda")] for a in range(3)], dim=1)  # (n, 64, 2)
    fidx = perm.forward_dev.long()

    def unfused():
        res = []
        for j in range(3):
            x = qkv[:, j][fidx].float()  # gather
            if j < 2:
                x0, x1 = x[..., 0::2], x[..., 1::2]
                c, s_ = cs[:, None, :, 0], cs[:, None, :, 1]
                x = torch.stack([x0 * c - x1 * s_, x0 * s_ + x1 * c], dim=-1).flatten(-2)
            outs[j][:, :n] = x.to(torch.bfloat16).permute(1, 0, 2)
        return res

    t2 = timed(unfused, reps=5)
    recs.append({"kernel": "same result, unfused torch (gather, rotate, cast, transpose)", "ms": round(t2, 4),
                 "speedup_of_fused": round(t2 / t, 2)})
    C = 16
    lat = torch.randn((33, 45, 80, C), device="cuda")
    vel = torch.randn((n, C), device="cuda")
    t = timed(lambda: fused.unpermute_euler(lat, vel, perm, 0.7, 0.6), reps=20)
    byts = 3 * lat.numel() * 4 + 4 * n
    recs.append({"kernel": "unpermute_euler (invert_permutation + Euler, one pass)", "shape": "(33,45,80,16) f32",
                 "ms": round(t, 4), "gbs": round(byts / (t * 1e-3) / 1e9, 1)})
    t = timed(lambda: fused.curve_positions(perm), reps=20)
    recs.append({"kernel": "curve_positions", "shape": "118800 x 3 int64", "ms": round(t, 4)})
    return recs


def c1_record():
    """C1: the reference's CPU-runnable case (8x16x16 + 64 text, H=4, d=64, m=64, fp32, the
    paper-default k=0.3/p=0.3): fp32 SIMT carve path (the 1e-5 parity path) + mask build."""
    dims = tcb.GridDims(8, 16, 16)
    lay = tcb.build_layout(dims, 64, 64)
    st = tcb.StaticMasks.build(lay, dims, tcb.build_curve(dims))
    rng = np.random.default_rng(0)
    q, k, v = (torch.from_numpy(rng.standard_normal((4, lay.padded_total, 64), dtype=np.float32)).cuda()
               for _ in range(3))
    prm = tcb.SelectionParams(k=0.3, p=0.3)
    mask, _ = tcb.build_block_mask(q, k, lay, st, prm)
    inp = tcb.AttentionInputs(q=q, k=k, v=v, layout=lay)
    t_mask = timed(lambda: tcb.build_block_mask(q, k, lay, st, prm))
    t_carve = timed(lambda: tcb.carve_attention(inp, mask))
    return {"config": "C1 8x16x16 + 64 text, H=4, d=64, m=64, fp32, k=0.3 p=0.3", "mask_ms": round(t_mask, 4),
            "carve_ms": round(t_carve, 4), "kept_fraction": round(mask.selected_fraction, 4),
            "note": "tiled fp32 kernel k_carve_f32t (fp32 inputs keep fp32 math for the 1e-5 parity); "
                    "latency-bound at this size; the reference takes 0.13-0.16 s (SURVEY §6)"}


def c2_fp32_record():
    """C2 with fp32 Q/K/V (the reference's dtype, what a numpy caller gets): the tensor-core
    split-fp16 carve (k_carve_x3, within 1e-5 of the reference) at full size."""
    g = tcb.GridDims(33, 45, 80)
    lay = tcb.build_layout(g, 128, 256)
    st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
    gen = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn((24, lay.padded_total, 128), generator=gen, device="cuda") for _ in range(3))
    prm = tcb.SelectionParams(k=0.08, p=0.0)
    mask, _ = tcb.build_block_mask(q, k, lay, st, prm)
    inp = tcb.AttentionInputs(q=q, k=k, v=v, layout=lay)
    t_mask = timed(lambda: tcb.build_block_mask(q, k, lay, st, prm), reps=3, warm=1)
    t_carve = timed(lambda: tcb.carve_attention(inp, mask), reps=3, warm=1)
    pairs = int(mask.kv_cnt.sum().item()) + 24 * lay.M_c * lay.M_total
    return {"config": "C2 with fp32 inputs (k_carve_x3: fp16 hi/lo split products, 1e-5)", "mask_ms": round(t_mask, 3),
            "carve_ms": round(t_carve, 3), "layer_ms": round(t_mask + t_carve, 3),
            "fp32_tflops": round(4.0 * 128 ** 3 * pairs / (t_carve * 1e-3) / 1e12, 1)}


def dense_library_record():
    """Dense attention over the whole C2 sequence (931^2 x 24 block pairs) with the vendor
    kernels on the same box: torch SDPA (cuDNN / flash backends) and flash_attn if present.
    The kept-block TFLOP/s of k_carve_tc is judged against what a production dense kernel
    reaches under the same power cap."""
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel

    N, H, d = 931 * 128, 24, 128
    flops = 4.0 * N * N * d * H
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn((1, H, N, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = []

    def timed(name, fn, reps=3):
        try:
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            out.append({"kernel": name, "ms": round(ms, 2), "tflops": round(flops / (ms * 1e-3) / 1e12, 1)})
        except Exception as e:  # backend not available for this shape / build
            out.append({"kernel": name, "unavailable": str(e).splitlines()[0][:120]})

    for name, be in (("sdpa cudnn", SDPBackend.CUDNN_ATTENTION), ("sdpa flash", SDPBackend.FLASH_ATTENTION)):
        def run(be=be):
            with sdpa_kernel([be]):
                F.scaled_dot_product_attention(q, k, v)
        timed(name, run)
    try:
        from flash_attn import flash_attn_func
        qt, kt, vt = (t.transpose(1, 2).contiguous() for t in (q, k, v))
        timed("flash_attn 2.8 (library)", lambda: flash_attn_func(qt, kt, vt))
    except ImportError:
        out.append({"kernel": "flash_attn", "unavailable": "not importable"})
    return {"shape": f"(1, {H}, {N}, {d}) bf16, no mask", "flops": flops, "results": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-sweep", action="store_true")
    a = ap.parse_args()
    res = {"device": torch.cuda.get_device_name(0), "hbm": hbm_records(), "c4_stage_switch": c4_records(),
           "fused_f1": fused_records()}
    res["c1"] = c1_record()
    res["c2_fp32"] = c2_fp32_record()
    res["c3"] = layer_record("C3 Wan2.1-14B 480p 21x30x52, H=40, no text", (21, 30, 52), 0, 40, 0.08)
    res["c2"] = layer_record("C2 HunyuanVideo 720p 33x45x80 + 256 text, H=24", (33, 45, 80), 256, 24, 0.08)
    # C4: the two stages of the stock 2-stage plan at 720p (cli.default_stage_plan: stage 1
    # is 33x34x60, k=0.3, beta from rho=0.5; stage 2 the target, k=0.2; p=0.3), with the
    # per-stage step counts of that plan (11 + 12 = 23 NFE)
    beta1 = tcb.compute_beta(33 * 34 * 60, 33 * 45 * 80, 0.5)
    s1 = layer_record("C4 stage 1 (0.75x): 33x34x60 + 256 text, H=24", (33, 34, 60), 256, 24, 0.3, 0.3, beta1)
    s2 = layer_record("C4 stage 2 (1x): 33x45x80 + 256 text, H=24", (33, 45, 80), 256, 24, 0.2, 0.3)
    res["c4_layers"] = {"stage1": s1, "stage2": s2, "nfe": [11, 12],
                        "attention_ms_per_layer_sum_over_nfe": round(11 * s1["layer_ms"] + 12 * s2["layer_ms"], 2),
                        "note": "x number of attention layers of the DiT (60 for HunyuanVideo-13B) for the "
                                "sampler's attention time; stage switch kernels in c4_stage_switch"}
    if not a.skip_sweep:
        res["c5_sweep"] = [layer_record("C5 sweep on C2", (33, 45, 80), 256, 24, k)
                           for k in (0.01, 0.02, 0.05, 0.08, 0.10, 0.20, 0.30)]
    # dense-FA roofline reference for C5: all 931^2 x 24 pairs at the measured bf16 peak
    _, tf = peaks()
    dense = 4.0 * 128 ** 3 * 931 ** 2 * 24
    res["c5_dense_roofline_ms"] = round(dense / (tf * 1e12) * 1e3, 3)
    res["c2_dense_library"] = dense_library_record()
    text = json.dumps(res, indent=1)
    print(text)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text + "\n")


if __name__ == "__main__":
    main()

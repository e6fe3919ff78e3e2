"""HBM-bound kernels of the path at their BASELINE.json sizes: CUDA-event timings (L2 flushed
before every timed launch) against the algorithmic bytes, and an ``--ncu`` mode that launches
each kernel once (after one warm-up) for an ``ncu --set full -k regex:...`` capture.

  python tools/prof_hbm.py [--out profiles/r02_hbm_kernels.json]
  ncu --set full --clock-control none --import-source on -k regex:'k_gather|k_upsample|k_rope|k_curve|k_adjacency|k_pool' \
      -o gpurun_out/r02_hbm python tools/prof_hbm.py --ncu

Algorithmic bytes: gather 2 n row_bytes + 4 n; pool 2 x (H N_pad d x 2) read
+ 2 x (H M_total d x 8) written; upsample_renoise src (+vel) read + eps read + dst written;
rope_permute 3 x (n H d x 2) read + 3 x (n H d x 2) written + the index; curve 8 n written.
"""

import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_16864_b200 as tcb  # noqa: E402
from paper_2505_16864_b200 import _native  # noqa: E402
from paper_2505_16864_b200.partition import mask_words  # noqa: E402


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


FLUSH = None


def flush():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
    FLUSH.fill_(1)


def timed(fn, reps):
    """median ms of `reps` launches, each timed alone after an L2 flush"""
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def kernels():
    """(name, shape, algorithmic bytes, launcher) for every HBM kernel of the path."""
    s = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    out = []
    dims = tcb.GridDims(33, 45, 80)
    perm = tcb.build_curve(dims)
    n = dims.n_cells
    x = torch.randn((n, 3072), device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    out.append(("k_gather (permute_rows, K2)", "118800 x 3072 bf16 (C2 hidden)",
                2 * x.numel() * 2 + 4 * n,
                lambda: tcb.gather_rows(x, perm.forward_dev, out=y)))
    lay = tcb.build_layout(dims, 128, 256)
    q = torch.randn((24, lay.padded_total, 128), device="cuda").to(torch.bfloat16)
    k = torch.randn_like(q)
    pq = torch.empty((24, lay.M_total, 128), dtype=torch.float64, device="cuda")
    pk = torch.empty_like(pq)
    out.append(("k_pool (block_pool Q+K, K3)", "2 x 24 x 119168 x 128 bf16 (C2)",
                2 * q.numel() * 2 + 2 * pq.numel() * 8,
                lambda: _native.call("tcb_block_pool", q.data_ptr(), k.data_ptr(), 1, q.stride(0),
                                     q.stride(1), 24, 128, 128, lay.M_v, lay.M_total, lay.n_valid,
                                     lay.n_cond, pq.data_ptr(), pk.data_ptr(), s())))
    # RoPE + permute: raster token-major (n, H, d) -> curve head-major (H, N_pad, d)
    src = [torch.randn((n, 24, 128), device="cuda").to(torch.bfloat16) for _ in range(3)]
    dst = [torch.empty((24, lay.padded_total, 128), dtype=torch.bfloat16, device="cuda")
           for _ in range(3)]
    tcb.fused.rope_tables(dims, device=src[0].device)
    out.append(("k_rope_permute (qkv_to_curve, f-1)", "3 x 118800 x 24 x 128 bf16 (C2)",
                2 * 3 * n * 24 * 128 * 2 + 4 * n,
                lambda: tcb.rope_permute(src, perm, dst, [True, True, False])))
    fwd = torch.empty(n, dtype=torch.int32, device="cuda")
    inv = torch.empty_like(fwd)
    out.append(("k_curve (build_curve, K1)", "33x45x80", 8 * n,
                lambda: _native.call("tcb_curve_build", 33, 45, 80, fwd.data_ptr(), inv.data_ptr(), s())))
    words = mask_words(lay.M_total)
    adja = torch.empty((lay.M_v, words), dtype=torch.int32, device="cuda")
    out.append(("k_adjacency (adjacency_mask, K6)", "33x45x80, m=128", 4 * n + adja.numel() * 4,
                lambda: _native.call("tcb_adjacency_build", inv.data_ptr(), 33, 45, 80, 128, lay.M_v,
                                     words, adja.data_ptr(), s())))
    # C4 stage switch: (33,34,60,16) -> (33,45,80,16) fp32
    srcd, dstd, C = (33, 34, 60), (33, 45, 80), 16
    xs = torch.randn((*srcd, C), device="cuda")
    vel = torch.randn_like(xs)
    eps = torch.randn((*dstd, C), device="cuda")
    o = torch.empty_like(eps)
    nb_src, nb_dst = xs.numel() * 4, o.numel() * 4
    out.append(("k_upsample_renoise (upsample_area_3d, mode 0)", "(33,34,60,16)->(33,45,80,16) f32 (C4)",
                nb_src + nb_dst,
                lambda: _native.call("tcb_upsample_renoise", xs.data_ptr(), None, None, o.data_ptr(),
                                     *srcd, *dstd, C, 0.0, 0, 0, 0, s())))
    out.append(("k_upsample_renoise (stage_transition, host eps)", "(33,34,60,16)->(33,45,80,16) f32 (C4)",
                nb_src + 2 * nb_dst,
                lambda: _native.call("tcb_upsample_renoise", xs.data_ptr(), None, eps.data_ptr(),
                                     o.data_ptr(), *srcd, *dstd, C, 0.899083, 1, 0, 0, s())))
    out.append(("k_upsample_renoise (switch_stage: predict_clean + transition)",
                "(33,34,60,16)->(33,45,80,16) f32 (C4)", 2 * nb_src + 2 * nb_dst,
                lambda: _native.call("tcb_upsample_renoise", xs.data_ptr(), vel.data_ptr(),
                                     eps.data_ptr(), o.data_ptr(), *srcd, *dstd, C, 0.899083, 1, 0,
                                     0, s())))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ncu", action="store_true", help="one warm-up + one launch per kernel")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ks = kernels()
    torch.cuda.synchronize()
    if a.ncu:
        for _, _, _, fn in ks:
            fn()
            torch.cuda.synchronize()
            flush()
            torch.cuda.synchronize()
            fn()
            torch.cuda.synchronize()
        return
    peak, src = hbm_peak()
    recs = []
    for name, shape, nbytes, fn in ks:
        ms = timed(fn, a.reps)
        gbs = nbytes / (ms * 1e-3) / 1e9
        recs.append({"kernel": name, "shape": shape, "algorithmic_bytes": nbytes,
                     "ms_median": round(ms, 5), "us": round(ms * 1e3, 2), "gbs": round(gbs, 1),
                     "frac_of_hbm": round(gbs / peak, 3)})
    doc = {"peak_hbm_gbs": peak, "peak_source": src, "timing": "CUDA events, median of "
           f"{a.reps} launches, each after a 512 MB L2 flush", "kernels": recs}
    txt = json.dumps(doc, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(txt + "\n")


if __name__ == "__main__":
    main()

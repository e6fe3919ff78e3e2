"""Every head of a BASELINE layer against the oracle (an exhaustive version of
tests/test_gpu_fullsize_configs.py's sampled whole heads, too slow for the test suite):
--config C2 (default: 720p, H=24, k=0.08, p=0, bf16, the bench's seed), C3 (Wan 480p, H=40,
no text), C4s1 (stage 1 of the 2-stage plan: 33x34x60 + 256 text, k=0.3, p=0.3 cutoff,
beta=0.284) or the C5 sweep endpoints on C2 (C5k01: k=0.01, C5k30: k=0.30).  For each head: the device mask vs the
oracle's mask (bit-exact expected) and the carve output of every q-block vs the oracle's fp32
carve on the device mask (north_star bf16 tolerance 2e-2 of max|ref|).  One JSON line per
head to --out, a summary line on stdout.

  python tools/exhaustive_parity.py --out gpurun_out/exhaustive_parity.jsonl
"""

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch
from threadpoolctl import threadpool_limits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402  (test infrastructure: the checker, never the thing measured)
import paper_2505_16864_b200 as tcb  # noqa: E402

M = D = 128


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--config", default="C2", choices=["C2", "C3", "C4s1", "C5k01", "C5k30"])
    ap.add_argument("--seed", type=int, default=1234)
    a = ap.parse_args()
    cfg = {"C2": ((33, 45, 80), 256, 24, 0.08, 0.0, 0.0),
           "C3": ((21, 30, 52), 0, 40, 0.08, 0.0, 0.0),
           "C4s1": ((33, 34, 60), 256, 24, 0.3, 0.3,
                    -0.5 * math.log((33 * 34 * 60) / (33 * 45 * 80)) + 0.0),
           "C5k01": ((33, 45, 80), 256, 24, 0.01, 0.0, 0.0),
           "C5k30": ((33, 45, 80), 256, 24, 0.30, 0.0, 0.0)}[a.config]
    dims, nc, H, kr, pc, beta = cfg
    g = tcb.GridDims(*dims)
    lay = tcb.build_layout(g, M, nc)
    perm = tcb.build_curve(g)
    st = tcb.StaticMasks.build(lay, g, perm)
    gen = torch.Generator(device="cuda").manual_seed(a.seed)
    q, k, v = (torch.randn((H, lay.padded_total, D), generator=gen, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=kr, p=pc),
                                   need_relevance=False)
    out = tcb.carve_attention(tcb.AttentionInputs(q=q, k=k, v=v, layout=lay), mask,
                              tcb.AmplifierBias(beta))
    torch.cuda.synchronize()
    L = oracle.layout_scalars(dims, M, nc)
    adja = oracle.adjacency(dims, oracle.curve_inverse(perm.forward), M, L["M_v"])
    ok = oracle.token_valid(L)
    workers = max(1, len(os.sched_getaffinity(0)))
    worst, mism, t0 = 0.0, 0, time.time()
    with open(a.out, "w") as fh:
        for h in range(H):
            qh, kh, vh = (t[h: h + 1].float().cpu().numpy() for t in (q, k, v))
            with threadpool_limits(limits=workers, user_api="blas"):
                bits, _ = oracle.block_mask(qh, kh, L, adja, kr, pc)
            got_bits = mask.bits_dev[h].cpu().numpy()
            n_diff = int((got_bits != bits[0]).sum())
            with threadpool_limits(limits=1, user_api="blas"):
                ref = oracle.carve(qh, kh, vh, got_bits[None], L, beta, workers=workers)[0]
            got = out[h].float().cpu().numpy()
            scale = np.abs(ref).max()
            err = np.abs(got - ref)
            rel = float(err.max() / scale)
            blk = err.reshape(lay.M_total, M, D).max(axis=(1, 2)) / scale
            rms = float(np.sqrt(np.mean((got[ok] - ref[ok]) ** 2)) / np.sqrt(np.mean(ref[ok] ** 2)))
            rec = {"config": a.config, "head": h, "mask_blocks": int(bits[0].size),
                   "mask_differing_blocks": n_diff, "kept": int(bits[0].sum()),
                   "carve_max_rel_err": rel, "carve_rms_rel_err": rms,
                   "cond_rows_max_rel_err": float(blk[lay.M_v:].max()) if lay.M_c else None,
                   "padding_rows_zero": bool(np.all(got[~ok] == 0.0))}
            fh.write(json.dumps(rec) + "\n")
            fh.flush()
            worst = max(worst, rel)
            mism += n_diff
            print(json.dumps(rec), flush=True)
    print(json.dumps({"summary": f"{a.config} all heads", "heads": H, "mask_differing_blocks_total": mism,
                      "carve_max_rel_err_worst": worst, "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()

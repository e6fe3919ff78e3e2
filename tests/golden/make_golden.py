"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports ``tokencarve`` 0.1.0 from ``/root/reference/pkg/src`` and writes
small ``.npz`` fixtures next to this file.  The fixtures are committed; the
GPU box never reads ``/root/reference``.  Inputs are regenerated from the
seeds stored in each fixture (numpy ``default_rng`` streams are stable), so
only outputs (or per-row fingerprints of large outputs) are stored.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import tokencarve as tc  # noqa: E402
from tokencarve import pipeline as tpl  # noqa: E402


def sha16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, sorted(arrays))


def qkv(seed, H, N, d):
    rng = np.random.default_rng(seed)
    return tuple(rng.standard_normal((H, N, d), dtype=np.float32) for _ in range(3))


def curves():
    small = [(t, h, w) for t in range(1, 7) for h in range(1, 7) for w in range(1, 7)]
    small += [(1, 1, 7), (5, 1, 1), (3, 5, 7), (8, 8, 8), (2, 9, 4), (16, 23, 17), (8, 16, 16),
              (1, 45, 80), (2, 30, 52), (3, 34, 60), (7, 3, 2)]
    fw = [tc.build_curve(tc.GridDims(*d)).forward for d in small]
    big = [(33, 45, 80), (32, 45, 80), (21, 30, 52), (33, 34, 60), (8, 16, 16), (40, 3, 61)]
    big_fw = [tc.build_curve(tc.GridDims(*d)).forward.astype("<i8") for d in big]
    save(
        "curves.npz",
        small_dims=np.array(small, dtype=np.int64),
        small_offsets=np.cumsum([0] + [len(f) for f in fw]).astype(np.int64),
        small_forward=np.concatenate(fw).astype(np.int64),
        big_dims=np.array(big, dtype=np.int64),
        big_sha=np.array([sha16(f) for f in big_fw]),
        big_head=np.stack([f[:64] for f in big_fw]).astype(np.int64),
        big_tail=np.stack([f[-64:] for f in big_fw]).astype(np.int64),
    )


def layouts_and_adjacency():
    cases = [((4, 4, 4), 8, 0), ((3, 3, 3), 4, 3), ((8, 16, 16), 64, 64), ((4, 10, 12), 8, 12),
             ((5, 7, 9), 16, 5), ((2, 9, 4), 4, 0), ((6, 6, 6), 32, 7), ((33, 45, 80), 128, 256),
             ((21, 30, 52), 128, 0), ((33, 34, 60), 128, 256)]
    rows = []
    adj_blobs = []
    for dims, m, nc in cases:
        g = tc.GridDims(*dims)
        lay = tc.build_layout(g, m, nc)
        rows.append([*dims, m, nc, lay.n_valid, lay.M_v, lay.M_c, lay.M_total, lay.padded_total,
                     lay.cond_start, lay.valid_len])
        perm = tc.build_curve(g)
        adja = tc.adjacency_mask(lay, g, perm)
        adj_blobs.append(np.packbits(adja, axis=None))
    save(
        "layouts.npz",
        rows=np.array(rows, dtype=np.int64),
        adj_offsets=np.cumsum([0] + [len(b) for b in adj_blobs]).astype(np.int64),
        adj_packed=np.concatenate(adj_blobs),
        counts_333_4_3=tc.build_layout(tc.GridDims(3, 3, 3), 4, 3).block_valid_counts.astype(np.int64),
        ptc=np.array([[n, m, *tc.padded_token_count(n, m)] for n, m in
                      [(118800, 128), (1, 1), (7, 3), (256, 128), (129, 128), (32760, 128)]],
                     dtype=np.int64),
    )


def masks():
    out = {}
    # (name, dims, m, n_cond, H, d, k, p, seed)
    cases = [
        ("c1", (8, 16, 16), 64, 64, 4, 64, 0.3, 0.3, 0),
        ("c1k08", (8, 16, 16), 64, 64, 4, 64, 0.08, 0.0, 0),
        ("small", (4, 6, 8), 16, 5, 2, 16, 0.3, 0.3, 7),
        ("tiny", (3, 3, 3), 4, 3, 3, 8, 0.5, 0.6, 11),
        ("nocond", (5, 7, 9), 16, 0, 2, 32, 0.1, 0.0, 5),
    ]
    meta = []
    for name, dims, m, nc, H, d, k, p, seed in cases:
        g = tc.GridDims(*dims)
        lay = tc.build_layout(g, m, nc)
        perm = tc.build_curve(g)
        st = tc.StaticMasks.build(lay, g, perm)
        q, kk, _ = qkv(seed, H, lay.padded_total, d)
        mask, R = tc.build_block_mask(q, kk, lay, st, tc.SelectionParams(k=k, p=p))
        pq = tc.block_pool(q, lay)
        out[f"{name}_R"] = R
        out[f"{name}_bits"] = np.packbits(mask.bits, axis=-1)
        out[f"{name}_pq"] = pq.values
        out[f"{name}_counts"] = pq.valid_counts.astype(np.int64)
        meta.append([*dims, m, nc, H, d, seed, k, p])
    out["meta"] = np.array(meta, dtype=np.float64)
    out["names"] = np.array([c[0] for c in cases])
    # hand traces (test_masks.py:144-163)
    traces = []
    for row, k, p in [([0.5, 0.3, 0.15, 0.05], 0.25, 0.3), ([0.5, 0.3, 0.15, 0.05], 0.25, 0.6),
                      ([0.5, 0.3, 0.15, 0.05], 1.0, 0.0), ([0.25, 0.25, 0.25, 0.25], 0.5, 0.0)]:
        R = np.array(row, dtype=np.float64).reshape(1, 1, 4)
        b = tc.importance_mask(R, tc.SelectionParams(k=k, p=p), 4)[0, 0]
        traces.append([*row, k, p, *b.astype(np.float64)])
    out["traces"] = np.array(traces)
    # random rows with ties and a heavy head, for select-given-R parity
    rng = np.random.default_rng(123)
    Rr = rng.random((3, 40, 57))
    Rr[:, :, 10:20] = 0.5
    Rr[0, :5, 30:] = 0.0
    Rr = Rr / Rr.sum(-1, keepdims=True)
    out["randR"] = Rr
    for k, p in [(0.1, 0.0), (0.3, 0.3), (0.05, 0.9), (1.0, 0.5)]:
        out[f"randR_bits_{k}_{p}"] = np.packbits(
            tc.importance_mask(Rr, tc.SelectionParams(k=k, p=p), 40), axis=-1)
    save("masks.npz", **out)


def attention():
    out = {}
    cases = [
        # name, dims, m, n_cond, H, d, k, p, beta, seed
        ("c1", (8, 16, 16), 64, 64, 4, 64, 0.3, 0.3, 0.0, 0),
        ("c1beta", (8, 16, 16), 64, 64, 4, 64, 0.08, 0.0, 0.2876820724517809, 0),
        ("small", (4, 6, 8), 16, 5, 2, 16, 0.3, 0.3, 0.0, 7),
        ("m128", (2, 16, 20), 128, 40, 2, 128, 0.2, 0.0, 0.5, 3),
        ("m128nc", (3, 9, 13), 128, 0, 3, 128, 0.3, 0.0, 0.0, 4),
        ("d64", (2, 16, 20), 128, 130, 2, 64, 0.2, 0.1, 0.25, 8),
    ]
    meta = []
    for name, dims, m, nc, H, d, k, p, beta, seed in cases:
        g = tc.GridDims(*dims)
        lay = tc.build_layout(g, m, nc)
        perm = tc.build_curve(g)
        st = tc.StaticMasks.build(lay, g, perm)
        q, kk, v = qkv(seed, H, lay.padded_total, d)
        mask, _ = tc.build_block_mask(q, kk, lay, st, tc.SelectionParams(k=k, p=p))
        o = tc.carve_attention(tc.AttentionInputs(q=q, k=kk, v=v, layout=lay), mask,
                               tc.AmplifierBias(beta))
        out[f"{name}_bits"] = np.packbits(mask.bits, axis=-1)
        # per-row fingerprints keep the fixture small
        out[f"{name}_rowsum"] = o.astype(np.float64).sum(-1)
        out[f"{name}_rowsq"] = (o.astype(np.float64) ** 2).sum(-1)
        out[f"{name}_head"] = o[:, :8].copy()
        meta.append([*dims, m, nc, H, d, seed, k, p, beta])
    out["meta"] = np.array(meta, dtype=np.float64)
    out["names"] = np.array([c[0] for c in cases])
    out["beta_kat"] = np.array([tc.compute_beta(5625, 10000, 0.5), tc.compute_beta(10, 10, 0.5),
                                tc.compute_beta(67320, 118800, 0.5)])
    save("attention.npz", **out)


def stage_switch():
    out = {}
    cases = [((2, 3, 4), (3, 5, 7), 3), ((1, 2, 2), (1, 4, 4), 1), ((4, 6, 5), (4, 8, 5), 2),
             ((3, 34, 60), (3, 45, 80), 4)]
    for i, (src, dst, C) in enumerate(cases):
        rng = np.random.default_rng(40 + i)
        x = rng.standard_normal((*src, C), dtype=np.float32)
        vel = rng.standard_normal((*src, C), dtype=np.float32)
        up = tpl.upsample_area_3d(x, tc.GridDims(*dst))
        sigma = 0.899083
        x0 = tpl.predict_clean(x, vel, sigma)
        g = np.random.default_rng(99)
        tr = tpl.stage_transition(x0, sigma, tc.GridDims(*dst), g)
        tr0 = tpl.stage_transition(x0, 0.0, tc.GridDims(*dst), np.random.default_rng(99))
        out[f"case{i}_src"] = np.array(src)
        out[f"case{i}_dst"] = np.array(dst)
        out[f"case{i}_up"] = up
        out[f"case{i}_tr"] = tr
        out[f"case{i}_tr0"] = tr0
        for ax, (s, d) in enumerate(zip(src, dst)):
            out[f"case{i}_w{ax}"] = tpl._axis_weights(s, d)
    out["n_cases"] = np.array(len(cases))
    save("stage.npz", **out)


def pipeline_run():
    """Toy-transformer end-to-end run (pipeline.py:304-439), small."""
    plan = tpl.StagePlan(
        stages=(tpl.StageConfig(dims=tc.GridDims(2, 4, 6), step_indices=(0, 3, 6), alpha=3.0,
                                k=0.3, rho=0.5),
                tpl.StageConfig(dims=tc.GridDims(2, 6, 8), step_indices=(6, 8, 9), alpha=5.0,
                                k=0.2)),
        base_T=10, block_size=8, n_cond_tokens=5, p=0.3)
    den = tpl.toy_transformer_denoiser(channels=2, n_heads=2, d_k=16, seed=1234)
    res = tpl.run_pipeline(plan, den, rng=0, channels=2)
    sig = [s["sigma"] for s in res.report["steps"]]
    spars = [s["effective_sparsity"] for s in res.report["steps"]]
    save("pipeline.npz", latent=res.latent, sigmas=np.array(sig), sparsity=np.array(spars),
         betas=np.array([s["beta"] for s in res.report["stages"]]))


def positions():
    """Curve-order positional metadata exactly as run_pipeline builds it
    (pipeline.py:333-337), captured from inside the reference loop for two stages, plus
    the same construction at the C2 grid (fingerprint)."""
    seen = {}
    base = tpl.toy_transformer_denoiser(channels=1, n_heads=1, d_k=8, seed=3)

    def spy(z, ctx):
        seen.setdefault(ctx.dims.as_tuple(), np.array(ctx.positions))
        return base(z, ctx)

    plan = tpl.StagePlan(
        stages=(tpl.StageConfig(dims=tc.GridDims(2, 4, 6), step_indices=(0, 5), alpha=3.0, k=0.3),
                tpl.StageConfig(dims=tc.GridDims(3, 5, 7), step_indices=(5, 8), alpha=3.0, k=0.3)),
        base_T=10, block_size=8, n_cond_tokens=0, p=0.3)
    tpl.run_pipeline(plan, spy, rng=0, channels=1)
    dims = (33, 45, 80)
    n = dims[0] * dims[1] * dims[2]
    coords = np.stack(np.unravel_index(np.arange(n), dims), axis=1).astype(np.int64)
    big = tc.apply_permutation(coords, tc.build_curve(tc.GridDims(*dims)))
    save("positions.npz", s0=seen[(2, 4, 6)], s1=seen[(3, 5, 7)], c2_sha=np.array(sha16(big.astype("<i8"))),
         c2_head=big[:64])


def cli_outputs():
    """Files and stdout of the reference CLI (cli.py) for small cases, to check the GPU
    front end's outputs byte for byte (formats) or within tolerance (attention)."""
    import contextlib
    import io
    import json

    from tokencarve import cli as tcli
    from tokencarve import tensorio as tio

    d = os.path.join(HERE, "cli")
    os.makedirs(d, exist_ok=True)

    def run(argv):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = tcli.main(argv)
        assert rc == 0, argv
        return buf.getvalue()

    with open(os.path.join(d, "order_3_4_5.txt"), "w") as fh:
        fh.write(run(["order", "--dims", "3,4,5"]))
    run(["order", "--dims", "3,4,5", "--binary", "--out", os.path.join(d, "order_3_4_5.tct")])
    run(["masks", "--dims", "4,8,8", "--block", "16", "--cond", "5", "--heads", "2", "--dk", "16",
         "--seed", "0", "--rate", "0.3", "--cutoff", "0.3", "--out", os.path.join(d, "mask.tcm"),
         "--stats", os.path.join(d, "mask_stats.json"), "--csv", os.path.join(d, "neighbors.csv")])
    lay = tc.build_layout(tc.GridDims(4, 8, 8), 16, 5)
    rng = np.random.default_rng(21)
    for name in ("q", "k", "v"):
        tio.write_tensor(os.path.join(d, f"{name}.tct"),
                         rng.standard_normal((2, lay.padded_total, 16), dtype=np.float32))
    run(["attend", "--q", os.path.join(d, "q.tct"), "--k", os.path.join(d, "k.tct"), "--v",
         os.path.join(d, "v.tct"), "--dims", "4,8,8", "--block", "16", "--cond", "5", "--mask",
         os.path.join(d, "mask.tcm"), "--beta", "0.3", "--out", os.path.join(d, "attend_out.tct"),
         "--report", os.path.join(d, "attend_report.json")])
    with open(os.path.join(d, "plan_33_45_80.json"), "w") as fh:
        fh.write(run(["plan", "--target", "33,45,80", "--cond", "256", "--seed", "3"]))
    with open(os.path.join(d, "plan_3stage.json"), "w") as fh:
        fh.write(run(["plan", "--target", "16,40,64", "--stages", "3", "--base-steps", "30",
                      "--keep", "12", "--rates", "0.3,0.25,0.2", "--denoiser", "toy-transformer"]))
    rows = [run(["analyze", "--dims", "33,45,80", "--strategy", "sfc"]),
            run(["analyze", "--dims", "33,45,80", "--strategy", "tiled", "--tile", "4,8,8"]),
            run(["analyze", "--dims", "21,30,52", "--strategy", "tiled", "--tile", "3,6,6",
                 "--block", "64"])]
    with open(os.path.join(d, "analyze_rows.txt"), "w") as fh:
        fh.write("".join(rows))
    plan = {"stages": [{"dims": [2, 4, 6], "steps": [0, 3, 6], "alpha": 3.0, "k": 0.3, "rho": 0.5},
                       {"dims": [2, 6, 8], "steps": [6, 8, 9], "alpha": 5.0, "k": 0.2}],
            "base_steps": 10, "block_size": 8, "cond_tokens": 0, "p": 0.3, "seed": 4,
            "denoiser": "gaussian", "denoiser_params": {"mu": 3.0, "s": 2.0}, "channels": 2}
    with open(os.path.join(d, "pipeline_plan.json"), "w") as fh:
        json.dump(plan, fh)
    run(["pipeline", "--plan", os.path.join(d, "pipeline_plan.json"), "--out",
         os.path.join(d, "pipeline_latent.tct"), "--report", os.path.join(d, "pipeline_report.json")])
    print("wrote cli/")


if __name__ == "__main__":
    curves()
    layouts_and_adjacency()
    masks()
    attention()
    stage_switch()
    pipeline_run()
    positions()
    cli_outputs()

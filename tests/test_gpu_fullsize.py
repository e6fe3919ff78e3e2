"""Parity at BASELINE.json's full C2 size (33x45x80 + 256 text, H=24, d=128, m=128):

* masks of sampled heads bit-exact vs the oracle (the reference's algorithm on the same
  bf16-valued inputs; pooled means are exact, R within float64 rounding);
* carve output of sampled (head, q-block) items -- including both condition q-blocks and
  the partial last vision block -- within the bf16 tolerance of the fp32 oracle;
* size-independent properties over the whole layer: permutation round trip, every row
  holds its diagonal / adjacency / condition columns and >= n_floor blocks, padded query
  rows exactly zero, each output row inside the convex hull (per dim) of its kept V rows
  (checked on the sampled rows), bitwise run-to-run determinism of the full layer.
"""

import numpy as np

from golden_io import host as _host
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_2505_16864_b200")

DIMS, M, NC, H, D = (33, 45, 80), 128, 256, 24, 128


@pytest.fixture(scope="module")
def c2():
    g = tcb.GridDims(*DIMS)
    lay = tcb.build_layout(g, M, NC)
    perm = tcb.build_curve(g)
    st = tcb.StaticMasks.build(lay, g, perm)
    gen = torch.Generator(device="cuda").manual_seed(2505)
    q, k, v = (torch.randn((H, lay.padded_total, D), generator=gen, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    params = tcb.SelectionParams(k=0.08, p=0.0)
    mask, R = tcb.build_block_mask(q, k, lay, st, params)
    out = tcb.carve_attention(tcb.AttentionInputs(q=q, k=k, v=v, layout=lay), mask)
    torch.cuda.synchronize()
    return dict(g=g, lay=lay, perm=perm, st=st, q=q, k=k, v=v, mask=mask, R=R, out=out,
                params=params, L=oracle.layout_scalars(DIMS, M, NC))


def test_c2_permutation_roundtrip_and_fingerprint(c2):
    g = tcb.GridDims(*DIMS)
    x = torch.randn((g.n_cells, 3072), device="cuda").to(torch.bfloat16)
    z = tcb.apply_permutation(x, c2["perm"])
    assert torch.equal(tcb.invert_permutation(z, c2["perm"]), x)
    assert np.array_equal(c2["perm"].forward_np, oracle.curve_forward(DIMS))


@pytest.mark.parametrize("head", [0, 11, 23])
def test_c2_masks_bit_exact_on_sampled_heads(c2, head):
    L = c2["L"]
    qh = c2["q"][head: head + 1].float().cpu().numpy()
    kh = c2["k"][head: head + 1].float().cpu().numpy()
    adja = oracle.adjacency(DIMS, oracle.curve_inverse(oracle.curve_forward(DIMS)), M, L["M_v"])
    bits, R = oracle.block_mask(qh, kh, L, adja, 0.08, 0.0)
    got = c2["mask"].bits[head].cpu().numpy()
    assert np.array_equal(got, bits[0])
    np.testing.assert_allclose(c2["R"][head].cpu().numpy(), R[0], rtol=1e-12, atol=0)


def test_c2_mask_row_properties(c2):
    lay, mask = c2["lay"], c2["mask"]
    bits = _host(mask.bits)  # (H, M_v, M_total)
    adja = c2["st"].adja
    n_floor = c2["params"].n_floor(lay.M_v)
    assert np.all(bits[:, :, lay.M_v:])  # condition columns (the text sink)
    assert np.all(bits[:, :, : lay.M_v] >= adja[None])  # 3D neighbours incl. the diagonal
    cnt = mask.kv_cnt.cpu().numpy()
    assert np.array_equal(cnt, bits.sum(axis=2))
    assert cnt.min() >= n_floor
    idx = mask.kv_idx.cpu().numpy()
    for h, r in ((0, 0), (7, 500), (23, lay.M_v - 1)):
        row = idx[h, r, : cnt[h, r]]
        assert np.all(np.diff(row) > 0) and np.array_equal(row, np.flatnonzero(bits[h, r]))


def test_c2_carve_sampled_items_vs_oracle(c2):
    L, lay = c2["L"], c2["lay"]
    items = [(0, 0), (0, lay.M_v - 1), (5, 463), (13, 100), (23, 928),
             (3, lay.M_v), (20, lay.M_v + 1)]  # incl. partial last block and both cond rows
    heads = sorted({h for h, _ in items})
    sub = {h: i for i, h in enumerate(heads)}
    q, k, v = (c2[n][heads].float().cpu().numpy() for n in ("q", "k", "v"))
    bits = c2["mask"].bits[heads].cpu().numpy()
    ref = oracle.carve(q, k, v, bits, L, 0.0, workers=8, items=[(sub[h], b) for h, b in items])
    got = c2["out"][heads].float().cpu().numpy()
    for h, b in items:
        rows = slice(b * M, (b + 1) * M)
        r, gq = ref[sub[h], rows], got[sub[h], rows]
        err = np.abs(gq - r).max() / max(np.abs(r).max(), 1e-30)
        assert err <= 2e-2, (h, b, err)  # north_star bf16 tolerance
        # convex hull per dim of the kept V rows (softmax weights are a convex combination)
        kept = np.flatnonzero(bits[sub[h], b]) if b < lay.M_v else np.arange(lay.M_total)
        vk = np.concatenate([v[sub[h], j * M:(j + 1) * M] for j in kept])
        valid = oracle.token_valid(L)[rows]
        assert np.all(gq[valid] <= vk.max(0) + 2e-2) and np.all(gq[valid] >= vk.min(0) - 2e-2)


def test_c2_padding_rows_zero_and_determinism(c2):
    lay = c2["lay"]
    out = c2["out"]
    ok = torch.from_numpy(np.array(lay.token_valid_mask)).cuda()
    assert torch.count_nonzero(out[:, ~ok]) == 0
    again = tcb.carve_attention(tcb.AttentionInputs(q=c2["q"], k=c2["k"], v=c2["v"], layout=lay),
                                c2["mask"])
    assert torch.equal(again, out)  # bitwise run to run (fixed kv order, no atomics in the math)


@pytest.mark.parametrize("p", [0.0, 0.3])
def test_large_grid_beyond_c2_masks_and_carve(p):
    # 64x90x160 + 77 text tokens (921,677 tokens, M_total = 7,201 blocks, one head, d = 64):
    # rows this long select with one warp per CTA (the sort buffers need ~150 KB), and at
    # p = 0.3 nearly every row falls through the slim top-512 pass to the full sort
    dims, m, nc, d = (64, 90, 160), 128, 77, 64
    g = tcb.GridDims(*dims)
    lay = tcb.build_layout(g, m, nc)
    perm = tcb.build_curve(g)
    st = tcb.StaticMasks.build(lay, g, perm)
    gen = torch.Generator(device="cuda").manual_seed(7202)
    q, k, v = (torch.randn((1, lay.padded_total, d), generator=gen, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    mask, R = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=0.02, p=p))
    out = tcb.carve_attention(tcb.AttentionInputs(q=q, k=k, v=v, layout=lay), mask)
    torch.cuda.synchronize()
    L = oracle.layout_scalars(dims, m, nc)
    assert L["M_total"] == lay.M_total == 7201
    qn, kn, vn = (t.float().cpu().numpy() for t in (q, k, v))
    adja = oracle.adjacency(dims, oracle.curve_inverse(perm.forward_np), m, L["M_v"])
    rows = np.r_[0:64, L["M_v"] - 64:L["M_v"]]  # oracle selection on sampled rows
    pq, _ = oracle.pool_blocks(qn, L)
    pk, _ = oracle.pool_blocks(kn, L)
    Rs = oracle.relevance_f64(pq[:, rows], pk, d)
    bits = oracle.union_bits(oracle.select_topk(Rs, 0.02, p, L["M_v"]), adja[rows], L["M_v"])
    got = mask.bits[0].cpu().numpy()[rows]
    assert np.array_equal(got, bits[0])
    np.testing.assert_allclose(R[0, rows].cpu().numpy(), Rs[0], rtol=1e-12, atol=0)
    items = [(0, 0), (0, 3000), (0, L["M_v"] - 1), (0, L["M_v"])]  # last = condition row
    ref = oracle.carve(qn, kn, vn, _host(mask.bits), L, 0.0, workers=4, items=items)
    got = out.float().cpu().numpy()
    for _, b in items:
        sl = slice(b * m, (b + 1) * m)
        err = np.abs(got[0, sl] - ref[0, sl]).max() / max(np.abs(ref[0, sl]).max(), 1e-30)
        assert err <= 2e-2, (b, err)

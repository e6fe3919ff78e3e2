"""GPU parity of the fused neighbours of the path (§8f-1) through the C ABI: each fused
kernel against the unfused reference-order composition (bitwise) and the oracle."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_2505_16864_b200")
from paper_2505_16864_b200 import fused  # noqa: E402


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 3, 5), (8, 16, 16), (5, 9, 13), (33, 45, 80)])
def test_curve_positions_bit_exact(dims):
    perm = tcb.build_curve(tcb.GridDims(*dims))
    pos = fused.curve_positions(perm).cpu().numpy()
    assert pos.dtype == np.int64
    assert np.array_equal(pos, oracle.curve_positions(dims))


@pytest.mark.parametrize("patch", [(1, 1, 1), (1, 2, 2), (2, 1, 3)])
def test_patchify_permute_and_unpermute_euler(patch):
    dims = (3, 5, 7)
    g = tcb.GridDims(*dims)
    perm = tcb.build_curve(g)
    C = 4
    rng = np.random.default_rng(11)
    lat = rng.standard_normal((dims[0] * patch[0], dims[1] * patch[1], dims[2] * patch[2], C),
                              dtype=np.float32)
    tok = fused.patchify_permute(torch.from_numpy(lat).cuda(), perm, patch).cpu().numpy()
    ref_tok = oracle.patchify(lat, dims, patch)[oracle.curve_forward(dims)]
    assert np.array_equal(tok, ref_tok)
    if patch == (1, 1, 1):  # == the reference's apply_permutation of the flattened latent
        ap = tcb.apply_permutation(lat.reshape(-1, C), perm)
        assert np.array_equal(tok, ap)
    vel = rng.standard_normal(tok.shape, dtype=np.float32)
    out = fused.unpermute_euler(lat, vel, perm, 0.7, 0.55, patch)
    inv = oracle.curve_inverse(oracle.curve_forward(dims))
    v_lat = oracle.unpatchify(vel[inv], dims, patch, C)
    ref = lat + np.asarray(0.55 - 0.7, dtype=np.float32) * v_lat  # pipeline.py:137
    assert np.array_equal(out, ref)
    if patch == (1, 1, 1):
        two = tcb.denoise_step(lat, tcb.invert_permutation(vel, perm).reshape(lat.shape), 0.7, 0.55)
        assert np.array_equal(out, two)
    with pytest.raises(tcb.DomainError):
        fused.unpermute_euler(lat, vel, perm, 0.5, 0.6, patch)


def test_switch_stage_curve_matches_two_pass():
    src, dst = tcb.GridDims(3, 4, 6), tcb.GridDims(3, 6, 8)
    perm = tcb.build_curve(src)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 4, 6, 2), dtype=np.float32)
    vel_c = rng.standard_normal((src.n_cells, 2), dtype=np.float32)
    for sigma in (0.899083, 0.0, 1.0, 0.3):
        a = fused.switch_stage_curve(x, vel_c, perm, sigma, dst, np.random.default_rng(7))
        vel = tcb.invert_permutation(vel_c, perm).reshape(x.shape)
        b = tcb.switch_stage(x, vel, sigma, dst, np.random.default_rng(7))
        assert np.array_equal(a, b), sigma


@pytest.mark.parametrize("sections", [(16, 56, 56), (32, 48, 48), (0, 64, 64)])
def test_rope_permute_vs_oracle(sections):
    dims = (4, 6, 10)
    g = tcb.GridDims(*dims)
    perm = tcb.build_curve(g)
    lay = tcb.build_layout(g, 128, 20)
    n, H, d = g.n_cells, 3, 128
    gen = torch.Generator().manual_seed(3)
    qkv = torch.randn((n, 3, H, d), generator=gen).to(torch.bfloat16).cuda()  # interleaved
    q, k, v = qkv[:, 0], qkv[:, 1], qkv[:, 2]
    cond = tuple(torch.randn((H, 20, d), generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
    oq, ok, ov = fused.qkv_to_curve(q, k, v, perm, lay, sections, 256.0, cond=cond)
    assert oq.shape == (H, lay.padded_total, d)
    fwd = oracle.curve_forward(dims)
    pos = oracle.curve_positions(dims)
    for src, got, rot in ((q, oq, True), (k, ok, True), (v, ov, False)):
        x = src.float().cpu().numpy()[fwd]  # (n, H, d) in curve order
        if rot:
            x = oracle.rope_apply(x, pos, sections, 256.0, dims)
        want = torch.from_numpy(np.ascontiguousarray(x.transpose(1, 0, 2))).to(torch.bfloat16)
        got_c = got.cpu()
        assert torch.equal(got_c[:, :n], want)  # same fp32 ops, RNE to bf16: bitwise
        assert torch.count_nonzero(got_c[:, n: lay.cond_start]) == 0  # padding rows zero
    for o, c in zip((oq, ok, ov), cond):
        assert torch.equal(o[:, lay.cond_start: lay.cond_start + 20], c)


def test_rope_permute_identity_and_norm():
    dims = (2, 3, 4)
    g = tcb.GridDims(*dims)
    perm = tcb.build_curve(g)
    x = torch.randn((g.n_cells, 2, 64)).to(torch.bfloat16).cuda()
    out = torch.empty((2, g.n_cells, 64), dtype=torch.bfloat16, device="cuda")
    fused.rope_permute([x], perm, [out], [False], (0, 32, 32))
    fwd = torch.from_numpy(oracle.curve_forward(dims)).cuda()
    assert torch.equal(out, x[fwd].permute(1, 0, 2))
    fused.rope_permute([x], perm, [out], [True], (0, 32, 32))
    n0 = x[fwd].float().norm(dim=-1).permute(1, 0)
    n1 = out.float().norm(dim=-1)
    assert torch.allclose(n0, n1, rtol=2e-2)  # rotations preserve the norm (bf16 rounding)
    with pytest.raises(tcb.DomainError):
        fused.rope_permute([x], perm, [out], [True], (0, 30, 30))


def test_curve_positions_match_reference_loop_fixture():
    import golden_io as gio

    g = gio.load("positions.npz")
    for dims, key in (((2, 4, 6), "s0"), ((3, 5, 7), "s1")):
        pos = fused.curve_positions(tcb.build_curve(tcb.GridDims(*dims))).cpu().numpy()
        assert np.array_equal(pos, g[key])
    big = fused.curve_positions(tcb.build_curve(tcb.GridDims(33, 45, 80))).cpu().numpy()
    assert np.array_equal(big[:64], g["c2_head"])


def test_torch_ops_eager_and_compiled_match_api():
    # torch.ops.tokencarve.* (opaque custom ops with fake impls) inside a compiled model
    # function give the same bits as the API calls
    from paper_2505_16864_b200 import torch_ops  # noqa: F401

    dims = tcb.GridDims(3, 16, 24)
    lay = tcb.build_layout(dims, 128, 40)
    st = tcb.StaticMasks.build(lay, dims, tcb.build_curve(dims))
    prm = tcb.SelectionParams(k=0.3, p=0.0)
    gen = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn((lay.padded_total, 64), generator=gen, device="cuda")
    w = torch.randn((3, 64, 2 * 128), generator=gen, device="cuda") * 0.1
    adja = st.packed(lay)
    args = (lay.m, lay.M_v, lay.M_total, lay.n_valid, lay.n_cond)

    def layer(x):
        q, k, v = (torch.einsum("nf,fhd->hnd", x, w[i].view(64, 2, 128)).to(torch.bfloat16).contiguous()
                   for i in range(3))
        bits, kv_cnt = torch.ops.tokencarve.block_mask(q, k, adja, *args, prm.n_floor(lay.M_v), 0.0)
        o = torch.ops.tokencarve.carve(q, k, v, bits, kv_cnt, *args, 0.0)
        return o.float().sum(dim=0), bits

    eager, bits = layer(x)
    # aot_eager traces the whole function through the fake impls (fullgraph: no graph
    # breaks at the custom ops) without inductor codegen, which takes minutes cold
    compiled, bits_c = torch.compile(layer, fullgraph=True, backend="aot_eager")(x)
    assert torch.equal(bits, bits_c)
    torch.testing.assert_close(compiled, eager, rtol=2e-2, atol=2e-2)
    q = torch.einsum("nf,fhd->hnd", x, w[0].view(64, 2, 128)).to(torch.bfloat16).contiguous()
    k = torch.einsum("nf,fhd->hnd", x, w[1].view(64, 2, 128)).to(torch.bfloat16).contiguous()
    m_api, _ = tcb.build_block_mask(q, k, lay, st, prm)
    assert torch.equal(m_api.words, bits)

"""Pin the CPU oracle (oracle/port.py) to the golden vectors produced by the
real reference package (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

import golden_io as gio
import oracle


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a.astype("<i8")).tobytes()).hexdigest()[:16]


def test_small_curves_bit_exact():
    n = 0
    for dims, fw in gio.small_curves():
        got = oracle.curve_forward(dims)
        assert np.array_equal(got, fw), dims
        n += 1
    assert n > 200


def test_big_curve_fingerprints():
    g = gio.load("curves.npz")
    for i, dims in enumerate(g["big_dims"]):
        fw = oracle.curve_forward(tuple(int(v) for v in dims))
        assert sha16(fw) == str(g["big_sha"][i]), dims
        assert np.array_equal(fw[:64], g["big_head"][i])
        assert np.array_equal(fw[-64:], g["big_tail"][i])


def test_survey_fingerprints():
    # SURVEY.md §8c fingerprints, measured with the reference
    assert oracle.curve_forward((8, 16, 16))[:6].tolist() == [0, 256, 272, 16, 17, 273]
    assert oracle.curve_forward((33, 45, 80))[:6].tolist() == [0, 3600, 3680, 80, 160, 3760]


def test_layout_and_adjacency():
    for dims, m, nc, row, adj in gio.layout_rows():
        L = oracle.layout_scalars(dims, m, nc)
        assert [L["n_valid"], L["M_v"], L["M_c"], L["M_total"], L["padded_total"],
                L["cond_start"]] == [int(v) for v in row[5:11]]
        inv = oracle.curve_inverse(oracle.curve_forward(dims))
        got = oracle.adjacency(dims, inv, m, L["M_v"])
        assert np.array_equal(got, adj), (dims, m)
    g = gio.load("layouts.npz")
    L = oracle.layout_scalars((3, 3, 3), 4, 3)
    assert np.array_equal(oracle.block_counts(L), g["counts_333_4_3"])


@pytest.mark.parametrize("case", [c[0] for c in gio.mask_cases()])
def test_masks(case):
    for name, P, g in gio.mask_cases():
        if name != case:
            continue
        L = oracle.layout_scalars(P["dims"], P["m"], P["n_cond"])
        q, k, _ = gio.qkv(P["seed"], P["H"], L["padded_total"], P["d"])
        pq, cnt = oracle.pool_blocks(q, L)
        np.testing.assert_allclose(pq, g[f"{name}_pq"], rtol=0, atol=1e-12)
        assert np.array_equal(cnt, g[f"{name}_counts"])
        inv = oracle.curve_inverse(oracle.curve_forward(P["dims"]))
        adja = oracle.adjacency(P["dims"], inv, P["m"], L["M_v"])
        bits, R = oracle.block_mask(q, k, L, adja, P["k"], P["p"])
        np.testing.assert_allclose(R, g[f"{name}_R"], rtol=1e-12, atol=1e-15)
        assert np.array_equal(bits, gio.unpack_bits(g[f"{name}_bits"], L["M_total"]))
        # selection is bit-exact given the reference's own R
        top = oracle.select_topk(g[f"{name}_R"], P["k"], P["p"], L["M_v"])
        assert np.array_equal(oracle.union_bits(top, adja, L["M_v"]),
                              gio.unpack_bits(g[f"{name}_bits"], L["M_total"]))


def test_select_traces_and_random_rows():
    g = gio.load("masks.npz")
    for tr in g["traces"]:
        R = tr[:4].reshape(1, 1, 4)
        got = oracle.select_topk(R, float(tr[4]), float(tr[5]), 4)[0, 0]
        assert got.tolist() == [bool(v) for v in tr[6:]]
    R = g["randR"]
    for key in [k for k in g if k.startswith("randR_bits_")]:
        _, _, kk, p = key.split("_")
        got = oracle.select_topk(R, float(kk), float(p), 40)
        assert np.array_equal(got, gio.unpack_bits(g[key], R.shape[-1])), key


@pytest.mark.parametrize("case", ["small", "c1", "c1beta", "m128nc"])
def test_carve(case):
    for name, P, g in gio.attention_cases():
        if name != case:
            continue
        L = oracle.layout_scalars(P["dims"], P["m"], P["n_cond"])
        q, k, v = gio.qkv(P["seed"], P["H"], L["padded_total"], P["d"])
        bits = gio.unpack_bits(g[f"{name}_bits"], L["M_total"])
        out = oracle.carve(q, k, v, bits, L, P["beta"], workers=4)
        np.testing.assert_allclose(out.astype(np.float64).sum(-1), g[f"{name}_rowsum"],
                                   rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose((out.astype(np.float64) ** 2).sum(-1), g[f"{name}_rowsq"],
                                   rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(out[:, :8], g[f"{name}_head"], rtol=1e-5, atol=1e-6)
        # and the dense two-pass restatement agrees on the same mask
        if L["padded_total"] <= 2200:
            dense = oracle.dense_reference(q, k, v, oracle.mask_to_bias(bits, L, P["beta"]),
                                           oracle.token_valid(L))
            np.testing.assert_allclose(out, dense, rtol=1e-5, atol=2e-5)


def test_beta_kat():
    g = gio.load("attention.npz")
    got = [oracle.beta_of(5625, 10000, 0.5), oracle.beta_of(10, 10, 0.5),
           oracle.beta_of(67320, 118800, 0.5)]
    assert got == g["beta_kat"].tolist()
    assert abs(got[0] - 0.2876820724) < 1e-9


def test_stage_switch():
    g = gio.load("stage.npz")
    for i in range(int(g["n_cases"])):
        src, dst = tuple(g[f"case{i}_src"]), tuple(int(v) for v in g[f"case{i}_dst"])
        for ax in range(3):
            np.testing.assert_array_equal(oracle.area_weights(int(src[ax]), dst[ax]),
                                          g[f"case{i}_w{ax}"])
        rng = np.random.default_rng(40 + i)
        C = g[f"case{i}_up"].shape[-1]
        x = rng.standard_normal((*src, C), dtype=np.float32)
        vel = rng.standard_normal((*src, C), dtype=np.float32)
        np.testing.assert_allclose(oracle.upsample_area(x, dst), g[f"case{i}_up"], rtol=0,
                                   atol=1e-6)
        x0 = x - np.float32(0.899083) * vel
        noise = np.random.default_rng(99).standard_normal((*dst, C), dtype=np.float32)
        np.testing.assert_allclose(oracle.transition(x0, 0.899083, dst, noise), g[f"case{i}_tr"],
                                   rtol=0, atol=1e-6)


# ----------------------------------------------------------------- §8f-1 neighbours
def test_oracle_positions_match_reference_loop():
    g = gio.load("positions.npz")
    assert np.array_equal(oracle.curve_positions((2, 4, 6)), g["s0"])
    assert np.array_equal(oracle.curve_positions((3, 5, 7)), g["s1"])
    big = oracle.curve_positions((33, 45, 80))
    import hashlib
    assert hashlib.sha256(big.astype("<i8").tobytes()).hexdigest()[:16] == str(g["c2_sha"])


def test_oracle_patchify_roundtrip_and_rope_properties():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((4, 6, 10, 3)).astype(np.float32)
    for patch in ((1, 1, 1), (2, 3, 5), (1, 2, 2)):
        dims = (4 // patch[0], 6 // patch[1], 10 // patch[2])
        tok = oracle.patchify(x, dims, patch)
        assert np.array_equal(oracle.unpatchify(tok, dims, patch, 3), x)
    assert np.array_equal(oracle.patchify(x, (4, 6, 10), (1, 1, 1)), x.reshape(-1, 3))
    # position 0 -> angle 0 -> identity; rotations preserve pair norms
    dims = (2, 3, 4)
    q = rng.standard_normal((24, 2, 16)).astype(np.float32)
    zero = np.zeros((24, 3), np.int64)
    assert np.array_equal(oracle.rope_apply(q, zero, (4, 6, 6), 256.0, dims), q)
    pos = oracle.curve_positions(dims)
    r = oracle.rope_apply(q, pos, (4, 6, 6), 256.0, dims)
    np.testing.assert_allclose((r[..., 0::2] ** 2 + r[..., 1::2] ** 2),
                               (q[..., 0::2] ** 2 + q[..., 1::2] ** 2), rtol=1e-5)

"""Property tests of the reference suite (tokencarve tests/test_masks.py, test_attention.py),
run against the B200 kernels with hypothesis-drawn shapes and seeds:

* pooling: constant blocks pool to the constant, padding never enters a mean
  (test_masks.py:36-88);
* selection: monotone in p and in k, heads independent (test_masks.py:183-202);
* carving: invariant to a permutation of the tokens inside a kv block
  (test_attention.py:182-194), the attention mass on condition keys is non-decreasing in
  beta (test_attention.py:197-211), every output row is a convex combination of its kept
  V rows (test_attention.py:158-179).

fp32 inputs run the fp32-math kernels (1e-5), bf16 the tcgen05 kernel (north_star bf16
tolerance)."""

import numpy as np

from golden_io import host as _host
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_2505_16864_b200")

SETTINGS = settings(max_examples=15, deadline=None,
                    suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])

dims_st = st.tuples(st.integers(1, 4), st.integers(2, 9), st.integers(2, 9))


def _setup(dims, m, n_cond):
    g = tcb.GridDims(*dims)
    lay = tcb.build_layout(g, m, n_cond)
    return lay, tcb.StaticMasks.build(lay, g, tcb.build_curve(g))


@SETTINGS
@given(dims=dims_st, m=st.sampled_from([4, 16]), n_cond=st.integers(0, 9), seed=st.integers(0, 2**31))
def test_pool_constant_and_padding_excluded(dims, m, n_cond, seed):
    lay, _ = _setup(dims, m, n_cond)
    rng = np.random.default_rng(seed)
    H, d = 2, 8
    x = rng.standard_normal((H, lay.padded_total, d)).astype(np.float32)
    valid = lay.token_valid_mask
    x_pad = x.copy()
    x_pad[:, ~valid] = 1e6  # padding content must not matter
    a = _host(tcb.block_pool(x, lay).values)
    b = _host(tcb.block_pool(x_pad, lay).values)
    assert np.array_equal(a, b)
    c = np.full_like(x, 3.25)
    pc = _host(tcb.block_pool(c, lay).values)
    counts = np.asarray(lay.block_valid_counts)
    assert np.all(pc[:, counts > 0] == 3.25)


@SETTINGS
@given(rows=st.integers(1, 6), cols=st.integers(2, 300), seed=st.integers(0, 2**31),
       k=st.floats(0.01, 1.0), p1=st.floats(0.0, 0.95), p2=st.floats(0.0, 0.95))
def test_selection_monotone_in_p_and_k(rows, cols, seed, k, p1, p2):
    rng = np.random.default_rng(seed)
    R = rng.dirichlet(np.full(cols, 0.5), size=(2, rows))
    lo, hi = sorted((p1, p2))
    a = tcb.importance_mask(R, tcb.SelectionParams(k=k, p=lo), cols)
    b = tcb.importance_mask(R, tcb.SelectionParams(k=k, p=hi), cols)
    assert np.all(b >= a)  # a larger cutoff keeps a superset
    k2 = min(1.0, k * 2)
    c = tcb.importance_mask(R, tcb.SelectionParams(k=k2, p=lo), cols)
    assert np.all(c >= a)  # a larger quota keeps a superset


@SETTINGS
@given(dims=dims_st, seed=st.integers(0, 2**31))
def test_heads_are_independent(dims, seed):
    lay, stt = _setup(dims, 16, 5)
    rng = np.random.default_rng(seed)
    q, k, v = (rng.standard_normal((3, lay.padded_total, 16)).astype(np.float32) for _ in range(3))
    params = tcb.SelectionParams(k=0.3, p=0.2)
    mask, _ = tcb.build_block_mask(q, k, lay, stt, params)
    out = tcb.carve_attention(tcb.AttentionInputs(q=q, k=k, v=v, layout=lay), mask)
    for h in range(3):
        m1, _ = tcb.build_block_mask(q[h:h + 1], k[h:h + 1], lay, stt, params)
        o1 = tcb.carve_attention(tcb.AttentionInputs(q=q[h:h + 1], k=k[h:h + 1], v=v[h:h + 1],
                                                     layout=lay), m1)
        assert np.array_equal(_host(m1.bits)[0], _host(mask.bits)[h])
        assert np.array_equal(o1[0], out[h])


@SETTINGS
@given(dims=dims_st, seed=st.integers(0, 2**31), dtype=st.sampled_from(["f32", "bf16"]))
def test_carve_invariant_to_permutation_inside_kv_blocks(dims, seed, dtype):
    m = 16 if dtype == "f32" else 128
    d = 16 if dtype == "f32" else 128
    lay, stt = _setup(dims, m, 7)
    rng = np.random.default_rng(seed)
    q, k, v = (rng.standard_normal((2, lay.padded_total, d)).astype(np.float32) for _ in range(3))
    mask, _ = tcb.build_block_mask(q, k, lay, stt, tcb.SelectionParams(k=0.4, p=0.0))
    # shuffle the valid tokens inside every block (keys and values together)
    perm = np.arange(lay.padded_total)
    valid = lay.token_valid_mask
    for b in range(lay.M_total):
        idx = np.arange(b * m, (b + 1) * m)
        idx = idx[valid[idx]]
        perm[idx] = rng.permutation(idx)
    kp, vp = k[:, perm], v[:, perm]
    if dtype == "bf16":
        to = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)  # noqa: E731
        o1 = tcb.carve_attention(tcb.AttentionInputs(q=to(q), k=to(k), v=to(v), layout=lay), mask)
        o2 = tcb.carve_attention(tcb.AttentionInputs(q=to(q), k=to(kp), v=to(vp), layout=lay), mask)
        o1, o2 = o1.float().cpu().numpy(), o2.float().cpu().numpy()
        tol = 2e-2 * max(np.abs(o1).max(), 1e-30)
    else:
        o1 = tcb.carve_attention(tcb.AttentionInputs(q=q, k=k, v=v, layout=lay), mask)
        o2 = tcb.carve_attention(tcb.AttentionInputs(q=q, k=kp, v=vp, layout=lay), mask)
        tol = 1e-5 * max(np.abs(o1).max(), 1e-30)
    assert np.abs(o1 - o2).max() <= tol


@SETTINGS
@given(dims=dims_st, seed=st.integers(0, 2**31), b1=st.floats(0.0, 3.0), b2=st.floats(0.0, 3.0))
def test_condition_mass_non_decreasing_in_beta(dims, seed, b1, b2):
    lay, stt = _setup(dims, 16, 9)
    rng = np.random.default_rng(seed)
    q, k = (rng.standard_normal((2, lay.padded_total, 16)).astype(np.float32) for _ in range(2))
    v = np.zeros_like(q)
    v[:, lay.M_v * lay.m:, 0] = 1.0  # channel 0 = attention mass on condition keys
    mask, _ = tcb.build_block_mask(q, k, lay, stt, tcb.SelectionParams(k=0.3, p=0.0))
    lo, hi = sorted((b1, b2))
    ins = tcb.AttentionInputs(q=q, k=k, v=v, layout=lay)
    a = tcb.carve_attention(ins, mask, tcb.AmplifierBias(lo))[:, : lay.n_valid, 0]
    b = tcb.carve_attention(ins, mask, tcb.AmplifierBias(hi))[:, : lay.n_valid, 0]
    assert np.all(b >= a - 1e-6)


@SETTINGS
@given(dims=dims_st, seed=st.integers(0, 2**31))
def test_output_rows_are_convex_combinations(dims, seed):
    lay, stt = _setup(dims, 128, 3)
    rng = np.random.default_rng(seed)
    q, k, v = (torch.from_numpy(rng.standard_normal((2, lay.padded_total, 64)).astype(np.float32))
               .cuda().to(torch.bfloat16) for _ in range(3))
    mask, _ = tcb.build_block_mask(q, k, lay, stt, tcb.SelectionParams(k=0.2, p=0.0))
    out = tcb.carve_attention(tcb.AttentionInputs(q=q, k=k, v=v, layout=lay), mask).float().cpu()
    bits = _host(mask.bits)
    vn = v.float().cpu().numpy()
    valid = lay.token_valid_mask
    m = lay.m
    for h in range(2):
        for qb in range(lay.M_total):
            kept = np.flatnonzero(bits[h, qb]) if qb < lay.M_v else np.arange(lay.M_total)
            cols = np.concatenate([np.arange(b * m, (b + 1) * m) for b in kept])
            vk = vn[h, cols[valid[cols]]]
            rows = np.arange(qb * m, (qb + 1) * m)
            rows = rows[valid[rows]]
            o = out[h, rows].numpy()
            assert np.all(o <= vk.max(0) + 2e-2) and np.all(o >= vk.min(0) - 2e-2)


@settings(max_examples=40, deadline=None)
@given(rows=st.integers(1, 5), cols=st.integers(2, 2000), seed=st.integers(0, 2**31),
       k=st.floats(0.001, 1.0), p=st.floats(1e-6, 0.999), ties=st.booleans(),
       alpha=st.sampled_from([0.05, 0.5, 5.0]))
def test_selection_matches_oracle_on_random_rows(rows, cols, seed, k, p, ties, alpha):
    # bit-exact selection vs the oracle over the register window, the whole-row register
    # sort and the warp-parallel prefix (with its exact-chain fallback)
    import oracle
    rng = np.random.default_rng(seed)
    R = rng.dirichlet(np.full(cols, alpha), size=(1, rows))
    if ties:  # quantised values: many exact ties, prefixes landing on round numbers
        R = np.round(R * 64) / 64
    got = tcb.importance_mask(R, tcb.SelectionParams(k=k, p=p), cols)
    assert np.array_equal(got, oracle.select_topk(R, k, p, cols))

"""The reference's own acceptance criteria (tokencarve tests/test_acceptance.py), run
against the B200 implementation: criteria 05 (mask-builder contract), 06 (adjacency ==
brute-force 26-neighbourhood scan), 07 (Gaussian-denoiser sampling moments through the
device pipeline), 08 (stage-transition contract), 09 (skip schedule) and 10 (FLOPs
accounting).  Criteria 02/03 live in test_gpu_parity.py; 04 (curve properties) is covered
by the bit-exact curve tests.  The brute-force oracle below is written independently of
both the library and oracle/ (like the reference's tests/oracles.py)."""

import itertools
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_2505_16864_b200")


def brute_adjacency(dims, forward, m):
    """All-pairs Chebyshev-1 scan over cells lifted to blocks (diagonal set, symmetric)."""
    t, h, w = dims
    n = t * h * w
    coords = np.array(np.unravel_index(np.arange(n), dims)).T.astype(np.int32)
    pos = np.empty(n, np.int64)
    pos[forward] = np.arange(n)
    blk = pos // m
    nb = int(blk.max()) + 1
    a = np.eye(nb, dtype=bool)
    for s in range(0, n, 512):
        sub = coords[s: s + 512]
        i, j = np.nonzero(np.abs(sub[:, None, :] - coords[None, :, :]).max(axis=2) <= 1)
        a[blk[s + i], blk[j]] = True
    return a | a.T


def test_criterion_05_mask_builder_contract():
    rng = np.random.default_rng(55)
    rows = 0
    for p in (0.0, 0.3, 0.5, 0.9):
        for _ in range(5):
            m_v = int(rng.integers(4, 40))
            m_total = m_v + int(rng.integers(0, 4))
            k = float(rng.choice([0.1, 0.25, 0.3]))
            r = rng.dirichlet(np.full(m_total, 0.6), size=(2, 40))
            bits = tcb.importance_mask(r, tcb.SelectionParams(k=k, p=p), m_v)
            assert ((r * bits).sum(axis=-1) > p).all()
            assert (bits.sum(axis=-1) >= math.ceil(k * m_v)).all()
            rows += r.shape[0] * r.shape[1]
    assert rows >= 1000
    row = np.array([[[0.5, 0.3, 0.15, 0.05]]])
    assert tcb.importance_mask(row, tcb.SelectionParams(k=0.25, p=0.3), 4)[0, 0].tolist() == \
        [True, False, False, False]
    assert tcb.importance_mask(row, tcb.SelectionParams(k=0.25, p=0.6), 4)[0, 0].tolist() == \
        [True, True, False, False]
    assert tcb.importance_mask(row, tcb.SelectionParams(k=1.0, p=0.0), 4)[0, 0].all()


def test_criterion_06_adjacency_equals_brute_force():
    big = [(16, 16, 16), (1, 64, 64), (64, 8, 8), (4, 32, 32), (3, 8, 16), (6, 8, 8), (2, 45, 40),
           (5, 7, 9), (12, 12, 12), (7, 11, 13), (1, 1, 128), (31, 2, 33)]
    for dims_t in list(itertools.product(range(1, 7), repeat=3)) + big:
        dims = tcb.GridDims(*dims_t)
        perm = tcb.build_curve(dims)
        fw = perm.forward_np
        for m in (4, 8, 16):
            lay = tcb.build_layout(dims, m)
            got = tcb.adjacency_mask(lay, dims, perm)
            assert np.array_equal(got, brute_adjacency(dims_t, fw, m)), (dims_t, m)


def test_criterion_07_gaussian_sampling_moments():
    dims = tcb.GridDims(22, 22, 22)
    den = tcb.gaussian_analytic_denoiser(mu=3.0, s=2.0)
    full = tcb.StagePlan(stages=(tcb.StageConfig(dims, tuple(range(50)), alpha=1.0, k=1.0),),
                         base_T=50, block_size=128)
    cells = tcb.run_pipeline(full, den, rng=7).latent.ravel()
    assert cells.size >= 10_000
    assert abs(float(cells.mean()) - 3.0) <= 0.05
    assert abs(float(cells.std()) - 2.0) <= 0.05 * 2.0
    skipped = tcb.StagePlan(
        stages=(tcb.StageConfig(dims, tuple(tcb.skip_schedule(50, 23)), alpha=1.0, k=1.0),),
        base_T=50, block_size=128)
    c23 = tcb.run_pipeline(skipped, den, rng=7).latent.ravel()
    assert abs(float(c23.mean()) - 3.0) <= 0.1
    assert abs(float(c23.std()) - 2.0) <= 0.1 * 2.0


def test_criterion_08_stage_transition_contract():
    rng = np.random.default_rng(88)
    x0 = rng.standard_normal((8, 50, 50, 5)).astype(np.float32)
    target = tcb.GridDims(8, 50, 50)
    pure = tcb.stage_transition(x0, 1.0, target, np.random.default_rng(3))
    assert abs(float(pure.mean())) <= 0.02 and abs(float(pure.std()) - 1.0) <= 0.02
    frozen = tcb.stage_transition(x0, 0.0, target, np.random.default_rng(3))
    assert frozen.tobytes() == tcb.upsample_area_3d(x0, target).tobytes()
    assert tcb.compute_beta(1234, 1234, 0.5) == 0.0
    assert abs(tcb.compute_beta(5625, 10000, 0.5) - 0.28768) <= 1e-5


def test_criterion_09_skip_schedule():
    idx = tcb.skip_schedule(50, 23)
    assert len(idx) == 23 and len(set(idx)) == 23 and idx[0] == 0 and idx[-1] == 49
    gaps = np.diff(idx)
    peak = int(np.argmax(gaps))  # unimodal: non-decreasing up to the peak, then non-increasing
    assert np.all(np.diff(gaps[: peak + 1]) >= 0) and np.all(np.diff(gaps[peak:]) <= 0)


def test_criterion_10_flops_accounting():
    rng = np.random.default_rng(1010)
    for _ in range(25):
        heads, rows = int(rng.integers(1, 5)), int(rng.integers(1, 12))
        cols = rows + int(rng.integers(0, 4))
        m, d_k = int(rng.choice([4, 16, 128])), int(rng.choice([8, 64]))
        bits = rng.random((heads, rows, cols)) < rng.uniform(0.05, 0.95)
        rep = tcb.attention_flops(tcb.BlockMask(bits=bits), m=m, d_k=d_k)
        assert rep.n_prime == m * int(bits.sum()) / (heads * rows)
    rep = tcb.attention_flops(tcb.BlockMask(bits=np.ones((3, 7, 9), bool)), m=16, d_k=32)
    assert rep.dense_ratio == 1.0 and rep.n_prime == 16 * 9

"""The p > 0 cutoff selection on raw scores (k_select_cut: no sort, rows of <= 1024 blocks)
against the reference algorithm applied to the very R values the device computed.

tcb_block_select_scores turns the pooled scores into R in place (every row) and selects;
tcb_block_mask selects from its own scratch.  Both must equal masks.py's importance_mask
(stable descending order, np.cumsum prefix, n_cut = #(prefix <= p) + 1, floor, cap) plus the
condition columns, restated here in numpy over that R -- on random, duplicated, near-tied,
flat and peaked rows, p from 0 (the R-returning p = 0 path) to 0.95, n_floor from 1 to M_v, widths around the kernel's
256 / 512 / 1024 splits and one beyond (the shared-memory path)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_2505_16864_b200")
from paper_2505_16864_b200 import _native  # noqa: E402
from paper_2505_16864_b200.partition import mask_words  # noqa: E402


def _pooled(H, M_total, d, kind, rng):
    pq = rng.standard_normal((H, M_total, d))
    pk = rng.standard_normal((H, M_total, d))
    if kind == "dups":
        src = rng.integers(0, M_total, M_total // 3)
        dst = rng.integers(0, M_total, M_total // 3)
        pk[:, dst] = pk[:, src]
    elif kind == "near":
        src = rng.integers(0, M_total, M_total // 4)
        pk[:, (src + 1) % M_total] = pk[:, src] * (1.0 + 1e-15)
    elif kind == "flat":
        pk[0] = pk[0, :1]
    elif kind == "peaked":  # R concentrated on a few columns: the cut lands early
        pq *= 3.0
    return pq, pk


def _ref_bits(R, n_floor, p, M_v):
    """masks.py:137-175 on R: importance_mask + condition columns (no adjacency)."""
    H, rows, n = R.shape
    order = np.argsort(-R, axis=-1, kind="stable")
    srt = np.take_along_axis(R, order, axis=-1)
    pre = np.cumsum(srt, axis=-1)
    n_cut = (pre <= p).sum(axis=-1) + 1
    keep = np.minimum(np.maximum(n_cut, n_floor), n)
    sel = np.arange(n) < keep[..., None]
    top = np.zeros(R.shape, dtype=bool)
    np.put_along_axis(top, order, sel, axis=-1)
    top[:, :, M_v:] = True
    return top


def _unpack(words_t, M_total):
    w = words_t.cpu().numpy().view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")
    return bits[..., :M_total].astype(bool)


@pytest.mark.parametrize("M_total", [40, 256, 300, 512, 700, 931, 1024, 1300])
@pytest.mark.parametrize("kind", ["random", "dups", "near", "flat", "peaked"])
def test_cutoff_select_equals_reference_on_device_R(M_total, kind):
    rng = np.random.default_rng(M_total * 11 + len(kind))
    H, d = 2, 64
    M_v = M_total - 2
    pq, pk = _pooled(H, M_total, d, kind, rng)
    pq_t, pk_t = torch.from_numpy(pq).cuda(), torch.from_numpy(pk).cuda()
    words = mask_words(M_total)
    st = torch.cuda.current_stream().cuda_stream
    for p in (0.0, 0.1, 0.3, 0.7, 0.95):
        for n_floor in sorted({1, max(1, M_total // 12), M_v}):
            S = torch.empty((H, M_v, M_total), dtype=torch.float64, device="cuda")
            _native.call("tcb_block_scores", pq_t.data_ptr(), M_total, pk_t.data_ptr(), H, M_v,
                         M_total, d, S.data_ptr(), st)
            b2 = torch.empty((H, M_v, words), dtype=torch.int32, device="cuda")
            c2 = torch.empty((H, M_v), dtype=torch.int32, device="cuda")
            _native.call("tcb_block_select_scores", S.data_ptr(), H, M_v, M_total, None, words,
                         n_floor, p, 1, b2.data_ptr(), c2.data_ptr(), st)  # S -> R in place
            bf = torch.empty_like(b2)
            cf = torch.empty_like(c2)
            scratch = torch.empty(max(H * M_v * M_total, M_total), dtype=torch.float64, device="cuda")
            _native.call("tcb_block_mask", pq_t.data_ptr(), M_total, pk_t.data_ptr(), H, M_v, M_total,
                         d, None, words, n_floor, p, bf.data_ptr(), cf.data_ptr(), scratch.data_ptr(),
                         scratch.numel(), st)
            torch.cuda.synchronize()
            want = _ref_bits(S.cpu().numpy(), n_floor, p, M_v)
            got2 = _unpack(b2, M_total)
            gotf = _unpack(bf, M_total)
            assert np.array_equal(got2, want), (kind, M_total, p, n_floor, int((got2 != want).sum()))
            assert np.array_equal(gotf, want), (kind, M_total, p, n_floor, int((gotf != want).sum()))
            assert np.array_equal(c2.cpu().numpy(), want.sum(axis=-1))
            assert np.array_equal(cf.cpu().numpy(), want.sum(axis=-1))

"""Differential test of the p == 0 register selection (k_select_p0, rows of <= 1024 blocks)
against the exact path on the same pooled scores: tcb_block_mask (scores into scratch, fast
top-n_floor on the scores, exact re-run of near-tie rows) must give bitwise the mask of
tcb_block_scores + tcb_block_select_scores (softmax in place, numpy's stable order) -- on
random rows, exact ties across the top-k boundary, near ties 1e-15 apart, n_floor from 1 to
M_total, and widths on both sides of the kernel's 256 / 512 / 1024 register splits."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_2505_16864_b200")
from paper_2505_16864_b200 import _native  # noqa: E402
from paper_2505_16864_b200.masks import mask_scratch  # noqa: E402
from paper_2505_16864_b200.partition import mask_words  # noqa: E402


def _pooled(H, M_total, d, kind, rng):
    pq = rng.standard_normal((H, M_total, d))
    pk = rng.standard_normal((H, M_total, d))
    if kind == "dups":  # exact score ties: duplicated key blocks
        src = rng.integers(0, M_total, M_total // 3)
        dst = rng.integers(0, M_total, M_total // 3)
        pk[:, dst] = pk[:, src]
    elif kind == "near":  # near ties: key blocks 1e-15 apart
        src = rng.integers(0, M_total, M_total // 4)
        pk[:, (src + 1) % M_total] = pk[:, src] * (1.0 + 1e-15)
    elif kind == "flat":  # every score equal in head 0
        pk[0] = pk[0, :1]
    return torch.from_numpy(pq).cuda(), torch.from_numpy(pk).cuda()


@pytest.mark.parametrize("M_total", [33, 200, 256, 257, 512, 513, 931, 1024, 1500])
@pytest.mark.parametrize("kind", ["random", "dups", "near", "flat"])
def test_fast_select_equals_exact_path(M_total, kind):
    rng = np.random.default_rng(M_total * 7 + len(kind))
    H, d = 3, 64
    M_v = M_total - 2
    pq, pk = _pooled(H, M_total, d, kind, rng)
    words = mask_words(M_total)
    st = torch.cuda.current_stream().cuda_stream
    for n_floor in sorted({1, 5, max(1, M_total // 12), M_v, M_total}):
        fast_bits = torch.empty((H, M_v, words), dtype=torch.int32, device="cuda")
        fast_cnt = torch.empty((H, M_v), dtype=torch.int32, device="cuda")
        scratch = torch.empty(max(H * M_v * M_total, M_total), dtype=torch.float64, device="cuda")
        _native.call("tcb_block_mask", pq.data_ptr(), M_total, pk.data_ptr(), H, M_v, M_total, d,
                     None, words, n_floor, 0.0, fast_bits.data_ptr(), fast_cnt.data_ptr(),
                     scratch.data_ptr(), scratch.numel(), st)
        S = torch.empty((H, M_v, M_total), dtype=torch.float64, device="cuda")
        _native.call("tcb_block_scores", pq.data_ptr(), M_total, pk.data_ptr(), H, M_v, M_total, d,
                     S.data_ptr(), st)
        ex_bits = torch.empty_like(fast_bits)
        ex_cnt = torch.empty_like(fast_cnt)
        _native.call("tcb_block_select_scores", S.data_ptr(), H, M_v, M_total, None, words, n_floor,
                     0.0, 1, ex_bits.data_ptr(), ex_cnt.data_ptr(), st)
        torch.cuda.synchronize()
        assert torch.equal(fast_cnt, ex_cnt), (kind, M_total, n_floor)
        assert torch.equal(fast_bits, ex_bits), (kind, M_total, n_floor)

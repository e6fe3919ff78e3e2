"""The tcgen05 carve kernel's condition-row split: with a full workspace each
condition q-block runs as kv-range chunks whose partials the last chunk merges; with a
256-byte workspace the same launch runs every condition row unsplit.  Vision rows never
split, so they must be bitwise identical either way; condition rows must agree with the
oracle within the bf16 tolerance, be run-to-run deterministic, and keep their padding rows
zero."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_2505_16864_b200")
from paper_2505_16864_b200 import _native  # noqa: E402
from paper_2505_16864_b200.attention import carve_work_bytes  # noqa: E402

BF16_GUARD = 1.4e-2  # as tests/test_gpu_parity.py


def _launch(q, k, v, mask, lay, beta, work_bytes):
    H, N, d = q.shape
    out = torch.empty_like(q)
    nb = max(work_bytes, 256)
    work = torch.zeros(nb, dtype=torch.uint8, device=q.device)
    _native.call("tcb_carve_fwd", q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), 1,
                 q.stride(0), q.stride(1), mask.words.data_ptr(), mask.words.shape[-1],
                 mask.kv_cnt.data_ptr(), H, d, 128, lay.M_v, lay.M_total, lay.n_valid, lay.n_cond,
                 float(beta), work.data_ptr(), work_bytes, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dims,n_cond,H,k_rate,beta", [
    ((4, 40, 60), 256, 3, 0.08, 0.0),     # M_total 77 + 2 text blocks: C = 1 (no split)
    ((8, 45, 80), 300, 2, 0.1, 0.3),      # M_total 228: C = 2, partial last text block
    ((12, 45, 80), 77, 2, 0.05, 0.0),     # 1 partial text block, C = 3
])
def test_split_condition_rows(dims, n_cond, H, k_rate, beta):
    gd = tcb.GridDims(*dims)
    lay = tcb.build_layout(gd, 128, n_cond)
    st = tcb.StaticMasks.build(lay, gd, tcb.build_curve(gd))
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    q, k, v = (torch.randn((H, lay.padded_total, 128), generator=g, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=k_rate, p=0.0),
                                   need_relevance=False)
    nb = carve_work_bytes(H, lay.M_v, lay.M_total, 128, 128)
    whole = _launch(q, k, v, mask, lay, beta, 256)
    split = _launch(q, k, v, mask, lay, beta, nb)
    again = _launch(q, k, v, mask, lay, beta, nb)
    vis = lay.M_v * 128
    assert torch.equal(split[:, :vis], whole[:, :vis])      # vision rows: untouched
    assert torch.equal(split, again)                         # deterministic merge order
    pad = torch.arange(lay.padded_total, device="cuda") >= lay.cond_start + lay.n_cond
    assert not split[:, pad].any()                           # condition padding rows zero
    qf, kf, vf = (t.float().cpu().numpy() for t in (q, k, v))
    L = oracle.layout_scalars(gd.as_tuple(), 128, n_cond)
    ref = oracle.carve(qf, kf, vf, mask.bits_dev.cpu().numpy(), L, beta, workers=8)
    cond = slice(vis, lay.padded_total)
    got = split[:, cond].float().cpu().numpy()
    err = np.abs(got - ref[:, cond]).max() / np.abs(ref[:, cond]).max()
    print(f"[bf16-err] split condition rows {dims}+{n_cond}: {err:.3e} (nbytes {nb})")
    assert err <= BF16_GUARD, err
    d_ws = (split[:, cond].float() - whole[:, cond].float()).abs().max().item()
    assert d_ws <= 2e-2 * np.abs(ref[:, cond]).max(), d_ws


def test_workspace_query():
    # no text -> no split (counter only); SIMT shapes -> counter only; C2 -> 8 chunks of 117
    assert carve_work_bytes(40, 256, 256, 128, 128) == 256
    assert carve_work_bytes(4, 32, 33, 64, 64) == 256
    nb = carve_work_bytes(24, 929, 931, 128, 128)
    assert nb == 256 + 256 + 24 * 2 * 8 * 128 * (128 + 2) * 4
    # a bounded workspace: 600 text blocks x 64 chunks x 24 heads would need ~30 GB -> unsplit
    assert carve_work_bytes(24, 7000, 7600, 128, 128) == 256

"""Where the carve kernel's DRAM traffic comes from: one carve launch per case for an ncu
capture of dram__bytes_read.sum (launch i of ``-k regex:k_carve_tc`` is case i):

  0  C2 (33x45x80 + 256, k=0.08), H=24       -- the bench layer
  1  C2, H=1                                 -- one head: no head transitions
  2  C2, H=24, no condition rows (n_cond=0)  -- no whole-head sweeps ahead of the vision rows
  3  C3 (21x30x52, no text), H=40            -- 16.8 MB of K/V per head

  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_carve_tc python tools/carve_l2_probe.py
Compulsory reads per case: Q + K + V once = 3 x H x N_pad x d x 2 bytes (printed).
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_16864_b200 as tcb  # noqa: E402
from paper_2505_16864_b200.attention import carve_raw  # noqa: E402


def case(dims, n_cond, H, k=0.08):
    gd = tcb.GridDims(*dims)
    lay = tcb.build_layout(gd, 128, n_cond)
    st = tcb.StaticMasks.build(lay, gd, tcb.build_curve(gd))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    q, kk, v = (torch.randn((H, lay.padded_total, 128), generator=g, device="cuda").to(torch.bfloat16)
                for _ in range(3))
    mask, _ = tcb.build_block_mask(q, kk, lay, st, tcb.SelectionParams(k=k, p=0.0),
                                   need_relevance=False)
    torch.cuda.synchronize()
    carve_raw(q, kk, v, mask, lay)
    torch.cuda.synchronize()
    pairs = int(mask.kv_cnt.sum().item()) + H * lay.M_c * lay.M_total
    print(f"dims={dims} n_cond={n_cond} H={H}: compulsory Q+K+V reads "
          f"{3 * H * lay.padded_total * 128 * 2 / 1e9:.3f} GB, K/V per head "
          f"{2 * lay.padded_total * 128 * 2 / 1e6:.1f} MB, kept pairs {pairs}", flush=True)


if __name__ == "__main__":
    case((33, 45, 80), 256, 24)
    case((33, 45, 80), 256, 1)
    case((33, 45, 80), 0, 24)
    case((21, 30, 52), 0, 40)

"""Small carve workload for instrumented ncu captures (source counters replay the kernel
~40 times; a full C2 layer would take minutes per pass).  Same C2 geometry and mask
statistics, fewer heads:

    ncu --set full --import-source on -k regex:k_carve_tc -s 2 -c 1 \
        python profiles/prof_carve.py --heads 2
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_16864_b200 as tcb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=2)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--k", type=float, default=0.08)
    a = ap.parse_args()
    dims = tcb.GridDims(33, 45, 80)
    lay = tcb.build_layout(dims, 128, 256)
    st = tcb.StaticMasks.build(lay, dims, tcb.build_curve(dims))
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    q, k, v = (torch.randn((a.heads, lay.padded_total, 128), generator=g, device="cuda")
               .to(torch.bfloat16) for _ in range(3))
    mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=a.k, p=0.0))
    out = torch.empty_like(q)
    for _ in range(a.iters):
        tcb.carve_raw(q, k, v, mask, lay, 0.0, out=out)
    torch.cuda.synchronize()
    print("ok", float(out.float().abs().mean()))


if __name__ == "__main__":
    main()

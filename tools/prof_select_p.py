"""Mask build at C2 with the paper-default cutoff (k=0.2, p=0.3): the p > 0 selection path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_16864_b200 as tcb

g = tcb.GridDims(33, 45, 80)
lay = tcb.build_layout(g, 128, 256)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
gen = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn((24, lay.padded_total, 128), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(2))
p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.3
for _ in range(3):
    m, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=0.2, p=p))
torch.cuda.synchronize()
print("kept", m.selected_fraction)

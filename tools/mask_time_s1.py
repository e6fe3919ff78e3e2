"""build_block_mask time at the C4 stage-1 geometry (33x34x60 + 256 text, H=24), p=0.3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_16864_b200 as tcb

g = tcb.GridDims(33, 34, 60)
lay = tcb.build_layout(g, 128, 256)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
gen = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn((24, lay.padded_total, 128), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(2))
for kk, p in ((0.3, 0.3), (0.3, 0.0)):
    prm = tcb.SelectionParams(k=kk, p=p)
    ts = []
    for i in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m, _ = tcb.build_block_mask(q, k, lay, st, prm)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[2:])
    print(f"stage1 k={kk} p={p}: mask {ts[len(ts)//2]:.3f} ms, kept {m.selected_fraction:.4f}")

"""One C2 fp32 carve layer (k_kv_absmax, k_kv_split, k_carve_x3) for ncu captures:
  ncu --set full --clock-control none -k regex:k_carve_x3 -c 1 -o gpurun_out/x3 python tools/prof_x3.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_16864_b200 as tcb

g = tcb.GridDims(33, 45, 80)
lay = tcb.build_layout(g, 128, 256)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
gen = torch.Generator(device="cuda").manual_seed(0)
H = int(os.environ.get("H", "24"))
q, k, v = (torch.randn((H, lay.padded_total, 128), generator=gen, device="cuda") for _ in range(3))
mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=0.08, p=0.0))
inp = tcb.AttentionInputs(q=q, k=k, v=v, layout=lay)
for _ in range(int(os.environ.get("REPS", "2"))):
    tcb.carve_attention(inp, mask)
torch.cuda.synchronize()
print("ok")

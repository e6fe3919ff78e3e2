"""e2e (pinned host Q/K/V -> O) layer time vs head-chunk size of carve_layer at C2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_16864_b200 as tcb

g = tcb.GridDims(33, 45, 80)
lay = tcb.build_layout(g, 128, 256)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
params = tcb.SelectionParams(k=0.08, p=0.0)
hq, hk, hv = (torch.randn((24, lay.padded_total, 128)).to(torch.bfloat16).pin_memory() for _ in range(3))
ho = torch.empty_like(hq).pin_memory()
for hpc in (1, 2, 3, 4, 6):
    for _ in range(2):
        tcb.carve_layer(hq, hk, hv, lay, st, params, out=ho, heads_per_chunk=hpc)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4):
        tcb.carve_layer(hq, hk, hv, lay, st, params, out=ho, heads_per_chunk=hpc)
    b.record()
    torch.cuda.synchronize()
    print("heads_per_chunk", hpc, round(a.elapsed_time(b) / 4, 2), "ms")
x = hq[:4].clone().pin_memory()
d = torch.empty(x.shape, dtype=x.dtype, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); d.copy_(x, non_blocking=True); b.record(); torch.cuda.synchronize()
print("H2D GB/s", round(x.numel() * 2 / a.elapsed_time(b) / 1e6, 1))

"""C2 carve time for bf16 vs fp16 inputs (same tcgen05 kernel, kind::f16 operand type)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_16864_b200 as tcb

g = tcb.GridDims(33, 45, 80)
lay = tcb.build_layout(g, 128, 256)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
for dt in (torch.bfloat16, torch.float16):
    gen = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn((24, lay.padded_total, 128), generator=gen, device="cuda").to(dt) for _ in range(3))
    mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=0.08, p=0.0))
    inp = tcb.AttentionInputs(q=q, k=k, v=v, layout=lay)
    for _ in range(3):
        tcb.carve_attention(inp, mask)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        tcb.carve_attention(inp, mask)
    b.record()
    torch.cuda.synchronize()
    print(dt, round(a.elapsed_time(b) / 10, 3), "ms")

"""A/B timing of the fused QKV RoPE permute at C2 (rotation on/off, token-major vs head-major source)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_16864_b200 as tcb
from paper_2505_16864_b200 import fused


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dims = tcb.GridDims(33, 45, 80)
perm = tcb.build_curve(dims)
lay = tcb.build_layout(dims, 128, 256)
n, H, d = dims.n_cells, 24, 128
qkv = torch.randn((n, 3, H, d), device="cuda").to(torch.bfloat16)
outs = [torch.zeros((H, lay.padded_total, d), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
srcs = [qkv[:, 0], qkv[:, 1], qkv[:, 2]]
byts = 2 * 3 * n * H * d * 2
for rot in ([True, True, False], [False, False, False]):
    t = timed(lambda: fused.rope_permute(srcs, perm, outs, rot))
    print("rotate", rot, f"{t:.4f} ms {byts / t / 1e6:.0f} GB/s")
sep = [torch.randn((n, H, d), device="cuda").to(torch.bfloat16) for _ in range(3)]
t = timed(lambda: fused.rope_permute(sep, perm, outs, [True, True, False]))
print("separate (n,H,d) sources", f"{t:.4f} ms {byts / t / 1e6:.0f} GB/s")
# write side alone: token-major destination (no transpose) via a plain gather of 6 KB rows
x = qkv[:, 0].contiguous()
y = torch.empty_like(x)
t = timed(lambda: tcb.gather_rows(x, perm.forward_dev, out=y))
print("gather_rows 6 KB rows", f"{t:.4f} ms {2 * x.numel() * 2 / t / 1e6:.0f} GB/s")

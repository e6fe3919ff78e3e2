"""Mask phase of the C2 layer: serial (pool all heads -> scores/select all heads) vs pipelined
over head chunks on two streams (pool of chunk c+1 on the main stream overlaps the
scores/select of chunk c on a side stream).  CUDA events, median of 20.  Masks compared
bitwise."""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_16864_b200 as tcb  # noqa: E402
from paper_2505_16864_b200 import _native  # noqa: E402
from paper_2505_16864_b200.masks import launch_mask, mask_buffers, mask_scratch  # noqa: E402

H, D, M = 24, 128, 128
g = tcb.GridDims(33, 45, 80)
lay = tcb.build_layout(g, M, 256)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
adja = st.packed(lay)
prm = tcb.SelectionParams(k=float(os.environ.get("K", "0.08")), p=float(os.environ.get("P", "0.0")))
gen = torch.Generator(device="cuda").manual_seed(1)
q, k = (torch.randn((H, lay.padded_total, D), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(2))
pq = torch.empty((H, lay.M_total, D), dtype=torch.float64, device="cuda")
pk = torch.empty_like(pq)
bits, cnt = mask_buffers(H, lay, "cuda")
scratch = mask_scratch(H, lay, "cuda")
main = torch.cuda.current_stream()
side = torch.cuda.Stream()


def pool(h0, h1, s):
    _native.call("tcb_block_pool", q[h0].data_ptr(), k[h0].data_ptr(), 1, q.stride(0), q.stride(1), h1 - h0,
                 D, M, lay.M_v, lay.M_total, lay.n_valid, lay.n_cond, pq[h0].data_ptr(), pk[h0].data_ptr(), s)


def serial():
    pool(0, H, main.cuda_stream)
    launch_mask(pq, pk, lay, adja, prm, bits, cnt, main.cuda_stream, scratch)


def piped(C):
    hc = H // C
    side.wait_stream(main)
    for c in range(C):
        h0, h1 = c * hc, (c + 1) * hc
        pool(h0, h1, main.cuda_stream)
        e = torch.cuda.Event()
        e.record(main)
        side.wait_event(e)
        launch_mask(pq[h0:h1], pk[h0:h1], lay, adja, prm, bits[h0:h1], cnt[h0:h1], side.cuda_stream, scratch)
    main.wait_stream(side)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


serial()
torch.cuda.synchronize()
ref_bits, ref_cnt = bits.clone(), cnt.clone()
print("serial", round(timed(serial), 4))
for C in (2, 3, 4, 6, 8, 12):
    t = timed(lambda: piped(C))
    same = torch.equal(bits, ref_bits) and torch.equal(cnt, ref_cnt)
    print("piped", C, round(t, 4), "bitwise" if same else "MISMATCH")

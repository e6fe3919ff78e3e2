"""CTA-0 timeline of the shipped carve kernel.  Needs a trace build:

    TCB_NVCC_EXTRA=-DTCB_CARVE_TRACE python -m paper_2505_16864_b200._build
    TCB_CARVE_DEBUG=8 python tools/carve_trace1.py     # 10 = also skip the softmax

(rebuild without TCB_NVCC_EXTRA afterwards; the stamps cost ~3 % when compiled in)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2505_16864_b200 as tcb
from paper_2505_16864_b200 import _native
EV, ST = 24, 8192
g = tcb.GridDims(33, 45, 80); lay = tcb.build_layout(g, 128, 256)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
gen = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((24, lay.padded_total, 128), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=0.08, p=0.0))
out = torch.empty_like(q)
lib = C.CDLL(_native.LIB_PATH); buf = (C.c_ulonglong * (EV * ST))()
for _ in range(2):
    tcb.carve_raw(q, k, v, mask, lay, 0.0, out=out); torch.cuda.synchronize()
    lib.tcb_debug_trace_read(buf, EV * ST)
T = np.frombuffer(buf, dtype=np.uint64).reshape(EV, ST).astype(np.int64)
base = T[T > 0].min(); T = np.where(T > 0, T - base, -1)
def d(e1, e0, s1=0, s0=0):
    n = ST - max(s1, s0); x1, x0 = T[e1][s1:s1 + n], T[e0][s0:s0 + n]
    m = (x1 >= 0) & (x0 >= 0); m[:3000] = False
    return float(np.median((x1 - x0)[m])) if m.any() else float("nan")
per = np.diff(T[5][T[5] >= 0]); print("half-step period (PV issued -> next)", np.median(per[3000:]))
print("MMA waits P", d(3, 1), "| PV issue", d(5, 3), "| K wait", d(8, 7), "| QK issue", d(9, 8))
print("softmax: waits S", d(10, 14), "| S seen -> P arrive", d(12, 10))
print("QK(t) issued -> S(t) seen", d(10, 9), "| P arrive -> MMA sees", d(3, 12))
rows = []
for e in range(EV):
    for i in range(5000, 5006):
        if T[e][i] >= 0: rows.append((T[e][i], e, i))
for c, e, i in sorted(rows): print(f"{c:>10d} ev{e:>3d} step{i:>5d}")

"""Read the carve kernel's CTA-0 pipeline timeline (TCB_CARVE_TRACE=1) and print per-block
latencies: MMA waits (K ready, P ready, V ready) and softmax phases."""
import ctypes
import os
import sys

import numpy as np

os.environ["TCB_CARVE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_16864_b200 as tcb  # noqa: E402
from paper_2505_16864_b200 import _native  # noqa: E402

lib = _native.load()
dims = tcb.GridDims(33, 45, 80)
lay = tcb.build_layout(dims, 128, 256)
st = tcb.StaticMasks.build(lay, dims, tcb.build_curve(dims))
g = torch.Generator(device="cuda"); g.manual_seed(0)
H = int(sys.argv[1]) if len(sys.argv) > 1 else 4
q, k, v = (torch.randn((H, lay.padded_total, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=0.08, p=0.0))
out = torch.empty_like(q)
buf = (ctypes.c_ulonglong * (8192 * 2))()
tcb.carve_raw(q, k, v, mask, lay, 0.0, out=out); torch.cuda.synchronize()
lib.tcb_debug_trace_read(buf, 8192)  # discard warm-up
tcb.carve_raw(q, k, v, mask, lay, 0.0, out=out); torch.cuda.synchronize()
n = lib.tcb_debug_trace_read(buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64)[: 2 * n].reshape(n, 2)
ev = (a[:, 0] >> 32).astype(int); step = (a[:, 0] & 0xffffffff).astype(int); clk = a[:, 1].astype(np.int64)
clk -= clk.min()
T = {}
for e, s_, c in zip(ev, step, clk):
    T.setdefault((e, s_), c)
names = {1: "mma:S issue", 2: "mma:K ready", 3: "mma:P ready", 4: "mma:V ready",
         12: "sm2:wait S", 22: "sm2:got S", 32: "sm2:P done", 19: "sm9:wait S", 29: "sm9:got S", 39: "sm9:P done"}
steps = sorted({s_ for (e, s_) in T if e == 3})
rows = []
for s_ in steps[5:200]:
    r = {nm: T.get((e, s_)) for e, nm in names.items()}
    rows.append(r)
def d(a_, b_):
    v = [r[b_] - r[a_] for r in rows if r[a_] is not None and r[b_] is not None]
    return np.median(v) if v else float("nan")
print("blocks traced", len(rows))
print("median sm2: got S -> P done (softmax compute)   ", d("sm2:got S", "sm2:P done"))
print("median sm9: got S -> P done                      ", d("sm9:got S", "sm9:P done"))
print("median sm2: wait S -> got S (waiting for S)      ", d("sm2:wait S", "sm2:got S"))
print("median mma: S issue -> K ready                   ", d("mma:S issue", "mma:K ready"))
print("median mma: P ready -> V ready                   ", d("mma:P ready", "mma:V ready"))
p = [T[(3, s_)] for s_ in steps]
print("median period between P ready (per block)        ", np.median(np.diff(p)))
print("median sm2 P done -> mma P ready (barrier lat)   ", d("sm2:P done", "mma:P ready"))
gs = sorted({s_ for (e, s_) in T if e == 22})
got = [T[(22, s_)] for s_ in gs]
print("median period between sm2 got S                  ", np.median(np.diff(got)))
# S(t) ready relative to P(t-1) ready
x = [T[(22, s_)] - T[(3, s_ - 1)] for s_ in gs if (3, s_ - 1) in T]
print("median sm2 got S(t) - mma P ready(t-1)           ", np.median(x))
y = [T[(1, s_)] - T[(3, s_ - 2)] for s_ in gs if (3, s_ - 2) in T and (1, s_) in T]
print("median mma S(t) issue - P ready(t-2)             ", np.median(y))

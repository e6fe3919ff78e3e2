"""Pipeline timeline of the two-tile carve kernel (CTA 0), TCB_CARVE_DEBUG bit 3.

    TCB_CARVE_V2=1 TCB_CARVE_DEBUG=8 python tools/carve_trace.py [--heads 24]

Per tile a, per global step: 1+a/3+a MMA before/after waiting P; 16+a V halves ready;
7+a/5+a MMA before/after the K halves of the next QK; 10+a/12+a softmax before/after
waiting S; 14+a P arrived.  Prints the median of each stage (cycles)."""

import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_16864_b200 as tcb  # noqa: E402
from paper_2505_16864_b200 import _native  # noqa: E402

EV, STEPS = 24, 4096


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--k", type=float, default=0.08)
    ap.add_argument("--dump", type=int, default=0)
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
    lib = C.CDLL(_native.LIB_PATH)
    buf = (C.c_ulonglong * (EV * STEPS))()
    tcb.carve_raw(q, k, v, mask, lay, 0.0, out=out)
    torch.cuda.synchronize()
    lib.tcb_debug_trace_read(buf, EV * STEPS)
    tcb.carve_raw(q, k, v, mask, lay, 0.0, out=out)
    torch.cuda.synchronize()
    lib.tcb_debug_trace_read(buf, EV * STEPS)
    T = np.frombuffer(buf, dtype=np.uint64).reshape(EV, STEPS).astype(np.int64)
    base = T[T > 0].min()
    T = np.where(T > 0, T - base, -1)

    def d(e1, e0, s1=0, s0=0):
        # median of T[e1][i+s1] - T[e0][i+s0] over steps where both exist (skip the first 50)
        a1, a0 = T[e1], T[e0]
        n = STEPS - max(s1, s0)
        x1, x0 = a1[s1:s1 + n], a0[s0:s0 + n]
        m = (x1 >= 0) & (x0 >= 0)
        m[:50] = False
        return float(np.median((x1 - x0)[m])) if m.any() else float("nan")

    for t in (0, 1):
        per = np.diff(T[12 + t][T[12 + t] >= 0])
        print(f"tile {t}: step period {np.median(per[50:]):.0f} | "
              f"softmax X (S seen -> P arrived) {d(14 + t, 12 + t):.0f} | "
              f"softmax idle (wait S) {d(12 + t, 10 + t):.0f} | "
              f"P arrived -> MMA sees P {d(3 + t, 14 + t):.0f} | "
              f"MMA waits P {d(3 + t, 1 + t):.0f} | MMA waits V {d(16 + t, 3 + t):.0f} | "
              f"MMA waits K {d(5 + t, 7 + t):.0f} | QK issued -> S seen {d(12 + t, 5 + t):.0f} | "
              f"PV issue {d(20 + t, 16 + t):.0f} | QK issue {d(18 + t, 5 + t):.0f}")
    if a.dump:
        rows = []
        for e in range(EV):
            for i in range(400, 400 + a.dump):
                if T[e][i] >= 0:
                    rows.append((T[e][i], e, i))
        for c, e, i in sorted(rows):
            print(f"{c:>10d} ev{e:>3d} step{i:>5d}")


if __name__ == "__main__":
    main()

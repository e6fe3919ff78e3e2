"""Error anatomy of the fp32 tensor-core carve (k_carve_x3) on one C2 head: max |err| / max |ref|
per row class (vision rows by kv-list length, condition rows) for x3 and the fp32 SIMT kernel."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2505_16864_b200 as tcb
from paper_2505_16864_b200.attention import carve_raw

dims, nc = (33, 45, 80), 256
g = tcb.GridDims(*dims)
lay = tcb.build_layout(g, 128, nc)
st = tcb.StaticMasks.build(lay, g, tcb.build_curve(g))
gen = torch.Generator(device="cuda").manual_seed(7)
q, k, v = (torch.randn((1, lay.padded_total, 128), generator=gen, device="cuda") for _ in range(3))
mask, _ = tcb.build_block_mask(q, k, lay, st, tcb.SelectionParams(k=float(os.environ.get("K", "0.08")), p=0.0))
x3 = carve_raw(q, k, v, mask, lay, 0.0).cpu().numpy()[0]
simt = carve_raw(q, k, v, mask, lay, 0.0, simt=True).cpu().numpy()[0]
L = oracle.layout_scalars(dims, 128, nc)
ref = oracle.carve(*(t.cpu().numpy() for t in (q, k, v)), mask.bits_dev.cpu().numpy(), L, 0.0, workers=16)[0]
den = np.abs(ref).max()
cnt = mask.kv_cnt.cpu().numpy()[0]
out = {"max_ref": float(den)}
for name, got in (("x3", x3), ("simt", simt)):
    e = np.abs(got - ref)
    rowerr = e.reshape(lay.M_total, 128, 128).max(axis=(1, 2))
    cls = {"cond": float(rowerr[lay.M_v:].max() / den)}
    for lo, hi in ((0, 60), (60, 100), (100, 200), (200, 1000)):
        sel = (cnt >= lo) & (cnt < hi)
        if sel.any():
            cls[f"vis_kv[{lo},{hi})"] = float(rowerr[:lay.M_v][sel].max() / den)
    # signed bias of the error on rows: mean(got - ref) / mean|ref|
    cls["mean_signed_rel"] = float((got - ref).mean() / np.abs(ref).mean())
    cls["rel_of_abs_scaled"] = float((np.abs(got) - np.abs(ref)).mean() / np.abs(ref).mean())
    out[name] = cls
print(json.dumps(out, indent=1))

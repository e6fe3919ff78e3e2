"""Diagnostic for the tcgen05 carve kernel on a single (head, q-block, kv-block):
prints the error against the correct result and against common layout mistakes
(V transposed, P transposed) so a wrong descriptor shows up by name."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_16864_b200 as tcb  # noqa: E402


def one_block(d=128, seed=0):
    dims = tcb.GridDims(1, 8, 16)  # 128 cells -> exactly one vision block
    lay = tcb.build_layout(dims, 128, 0)
    rng = np.random.default_rng(seed)
    q, k, v = (rng.standard_normal((1, 128, d), dtype=np.float32) for _ in range(3))
    qb, kb, vb = (torch.from_numpy(a).cuda().to(torch.bfloat16) for a in (q, k, v))
    mask = tcb.BlockMask(bits=np.ones((1, 1, 1), bool))
    out = tcb.carve_attention(tcb.AttentionInputs(q=qb, k=kb, v=vb, layout=lay), mask)
    torch.cuda.synchronize()
    o = out.float().cpu().numpy()[0]
    Q, K, V = (t.float().cpu().numpy()[0] for t in (qb, kb, vb))
    S = Q @ K.T / np.sqrt(d)
    P = np.exp(S - S.max(1, keepdims=True))
    P /= P.sum(1, keepdims=True)
    hyp = {"correct": P @ V, "P^T V": P.T @ V}
    if d == 128:
        hyp["P V^T"] = P @ V.T
    S2 = K @ Q.T / np.sqrt(d)
    P2 = np.exp(S2 - S2.max(1, keepdims=True)); P2 /= P2.sum(1, keepdims=True)
    hyp["S transposed"] = P2 @ V
    print(f"d={d}: nan={np.isnan(o).any()} |o|max={np.abs(o).max():.3f}")
    for name, h in hyp.items():
        print(f"   err vs {name:14s}: {np.abs(o - h).max():.4e}")
    return np.abs(o - hyp["correct"]).max()


if __name__ == "__main__":
    e1 = one_block(128)
    e2 = one_block(64)
    print("DIAG", "OK" if max(e1, e2) < 2e-2 else "FAIL")

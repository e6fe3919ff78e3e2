"""The reference's toy-transformer pipeline at the C4 720p 2-stage geometry on the device
(fp32, d_k=16 toy heads): wall time per NFE."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_16864_b200 as tcb
from paper_2505_16864_b200.cli import default_stage_plan

plan = default_stage_plan(tcb.GridDims(33, 45, 80), cond_tokens=256)
den = tcb.toy_transformer_denoiser(channels=16, n_heads=2, d_k=16)
t0 = time.perf_counter()
res = tcb.run_pipeline(plan, den, rng=0, channels=16)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"C4 toy pipeline: {plan.n_evaluations} NFE, {dt:.2f} s total, {dt / plan.n_evaluations * 1e3:.1f} ms/NFE")
print([round(s["effective_sparsity"], 3) for s in res.report["steps"]][:4], res.latent.shape)

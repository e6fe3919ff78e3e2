"""Benchmark: ms per carved-attention layer at HunyuanVideo 720p (BASELINE.json).

One step = one carved-attention layer on synthetic bf16 Q/K/V of the C2 shape
(33x45x80 = 118,800 video + 256 text tokens, H=24, d=128, m=128, k=0.08, p=0):
K3 block pool (Q,K) -> K4 pooled relevance -> K5 select/union -> K7/K8 carve.
With --gpus N>1 (torchrun) the layer is head-parallel: all-to-all (seq -> head
shard), the local layer on H/N heads, all-to-all back; value = max over ranks.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference itself
(tokencarve 0.1.0, pure numpy, installed unmodified into baseline/_ref) on the
box's host cores -- its build_block_mask over all heads plus its carve body on
consecutive slices of the layer's (head, q-block) jobs -- and prints the same
metric (the oracle port stands in only when baseline/_ref is absent).
"""

from __future__ import annotations

import argparse
import datetime
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# C2
DIMS = (33, 45, 80)
M = 128
N_COND = 256
H = 24
D = 128
K_RATE = 0.08
P_CUT = 0.0
METRIC = "ms per carved-attention layer at HunyuanVideo 720p"
WORKLOAD = ("C2 HunyuanVideo-13B attention layer: 720p 33x45x80=118,800 video + 256 text tokens, "
            "H=24, d=128, m=128 blocks (M_total=931), k=0.08 p=0 (~10% kept), bf16")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi sampler (every 50 ms) started before the warm-up, so that it is already
    producing when the timed region begins; only the samples whose timestamps fall inside
    the timed region (host clock, marked around the barriers) are summarised -- the nearest
    earlier sample stands in when the region is shorter than one sampling period."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None
        self.result = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            return None
        rows = []
        for line in out.strip().splitlines():
            r = line.split(", ")
            if len(r) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(r[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(r[1]), float(r[2]), r[3], r[4:8]))
            except ValueError:
                continue
        if not rows:
            return None
        inside = [r for r in rows if self.t0 is not None and self.t0 <= r[0] <= self.t1]
        if not inside:  # region shorter than a sampling period: the last sample before its end
            before = [r for r in rows if self.t1 is not None and r[0] <= self.t1]
            inside = before[-1:] or rows[-1:]
        sm = [r[1] for r in inside]
        mx = max(r[2] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i in range(4) if r[4][i].strip() == "Active"})
        pw = []
        for r in inside:
            try:
                pw.append(float(r[3]))
            except ValueError:
                pass
        self.result = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons,
                       "samples": len(inside),
                       "window_s": round(self.t1 - self.t0, 3) if self.t0 and self.t1 else None,
                       "power_w_median": statistics.median(pw) if pw else None}
        return self.result


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2505_16864_b200 as tcb
    from paper_2505_16864_b200 import _native
    from paper_2505_16864_b200.attention import _workspace, carve_work_bytes
    from paper_2505_16864_b200.masks import mask_scratch, launch_mask, mask_buffers
    from paper_2505_16864_b200.partition import mask_words

    world, rank, local = dist_env()
    # --dist-backend gloo: orchestration test with several ranks sharing the visible GPUs
    # (the exchange is staged through the host); production runs use NCCL, one GPU per rank
    local = local % torch.cuda.device_count() if args.dist_backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    _native.load()

    dims = tcb.GridDims(*DIMS)
    layout = tcb.build_layout(dims, M, N_COND)
    perm = tcb.build_curve(dims)
    statics = tcb.StaticMasks.build(layout, dims, perm)
    adja = statics.packed(layout)
    params = tcb.SelectionParams(k=K_RATE, p=P_CUT)
    Np, Mt, Mv = layout.padded_total, layout.M_total, layout.M_v
    Hl = H // world
    words = mask_words(Mt)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    if world == 1:
        # head-major (H, N, d) bf16, the layout carve_attention takes
        q, k, v = (torch.randn((H, Np, D), generator=g, device=dev, dtype=torch.float32)
                   .to(torch.bfloat16) for _ in range(3))
    else:
        n_loc = Np // world
        q, k, v = (torch.randn((n_loc, H, D), generator=g, device=dev, dtype=torch.float32)
                   .to(torch.bfloat16) for _ in range(3))

    pq = torch.empty((Hl, Mt, D), dtype=torch.float64, device=dev)
    pk = torch.empty_like(pq)
    bits, kv_cnt = mask_buffers(Hl, layout, dev)
    scratch = mask_scratch(Hl, layout, dev)
    work = _workspace(dev, carve_work_bytes(Hl, Mv, Mt, M, D))
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def layer(qh, kh, vh, out, marks=None, h0=0):
        """The launches of one carved-attention layer on head-major views (pool; scores into
        the bounded scratch + select/union on them -- a second select pass only re-runs
        near-tie rows; carve); mask buffers are used from local head h0 on (an exchange
        chunk's slice)."""
        sh, sn = qh.stride(0), qh.stride(1)
        Hc = qh.shape[0]  # all local heads, or one exchange chunk of them
        bq, bk = pq[h0:h0 + Hc], pk[h0:h0 + Hc]
        bb, bc = bits[h0:h0 + Hc], kv_cnt[h0:h0 + Hc]
        if marks: marks[0].record()
        _native.call("tcb_block_pool", qh.data_ptr(), kh.data_ptr(), 1, sh, sn, Hc, D, M, Mv, Mt,
                     layout.n_valid, layout.n_cond, bq.data_ptr(), bk.data_ptr(), sptr)
        if marks: marks[1].record()
        launch_mask(bq, bk, layout, adja, params, bb, bc, sptr, scratch)
        if marks: marks[2].record()
        _native.call("tcb_carve_fwd", qh.data_ptr(), kh.data_ptr(), vh.data_ptr(), out.data_ptr(), 1,
                     sh, sn, bb.data_ptr(), words, bc.data_ptr(), Hc, D, M, Mv, Mt, layout.n_valid,
                     layout.n_cond, 0.0, work.data_ptr(), work.numel(), sptr)
        if marks: marks[3].record()
        return out

    if world == 1:
        o = torch.empty_like(q)

        def step(marks=None):
            return layer(q, k, v, o, marks)
    else:
        from paper_2505_16864_b200.ulysses import carve_layer_sp, default_chunks, to_exchange_layout

        # token shards held in the exchange layout (C, G, n_loc, hc, d): the collectives send
        # and receive them without repacking (ulysses.py); converted once, outside the loop
        if args.a2a_chunks is None:
            args.a2a_chunks = default_chunks(Hl)
        C = args.a2a_chunks
        q, k, v = (to_exchange_layout(t, world, C) for t in (q, k, v))
        chunk = [0]

        def local(qh, kh, vh, _lay, out):
            h0 = chunk[0] * qh.shape[0]  # mask buffers of this chunk's heads
            chunk[0] += 1
            layer(qh, kh, vh, out, h0=h0)

        def step(marks=None):
            chunk[0] = 0
            if marks:  # per-kernel marks do not separate the exchange: time the whole layer
                marks[0].record()
            r = carve_layer_sp(q, k, v, layout, local, chunks=C)
            if marks:
                for mk in marks[1:]:
                    mk.record()
            return r

    red_dev = "cpu" if args.dist_backend == "gloo" else dev  # device of the scalar reductions

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clk = Clocks(local).start()  # sampling before the timed region starts (see Clocks)
    for _ in range(args.warmup):
        step()
    barrier()
    # kept pairs (algorithmic FLOPs = 4 m^2 d per kept (head, q-block, kv-block))
    pairs_local = int(kv_cnt.sum().item()) + Hl * layout.M_c * Mt
    pairs = pairs_local
    if world > 1:
        t = torch.tensor([pairs_local], device=red_dev, dtype=torch.int64)
        dist.all_reduce(t)
        pairs = int(t.item())

    marks = [[ev() for _ in range(4)] for _ in range(args.steps)]
    t0, t1 = ev(), ev()
    barrier()
    clk.mark_start()
    t0.record()
    for i in range(args.steps):
        step(marks[i])
    t1.record()
    barrier()
    clk.mark_end()
    clk.stop()
    total_ms = t0.elapsed_time(t1)
    per = np.array([[marks[i][j].elapsed_time(marks[i][j + 1]) for j in range(3)]
                    for i in range(args.steps)])
    ms_step = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    k_pool, k_sel, k_carve = per.mean(axis=0)
    chunked = world > 1
    if chunked:  # per-kernel marks do not separate the pipelined chunks: use the layer time
        k_pool = k_sel = float("nan")
        k_carve = ms_step
    flops = 4.0 * M * M * D * pairs
    flops_local = 4.0 * M * M * D * pairs_local
    hbm, tf_burst, tf_sust, peak_src = peaks()
    carve_tflops = flops_local / (k_carve * 1e-3) / 1e12

    # the same layer replayed as one CUDA graph (tcb.CarveLayerGraph): launch overhead gone
    graph_ms = None
    if world == 1:
        lg = tcb.CarveLayerGraph(q, k, v, layout, statics, params)
        for _ in range(2):
            lg.replay()
        barrier()
        a, b = ev(), ev()
        a.record()
        for _ in range(args.steps):
            lg.replay()
        b.record()
        barrier()
        graph_ms = round(a.elapsed_time(b) / args.steps, 4)
        del lg

    # e2e through the public API with host buffers (pinned H2D in, O D2H out)
    e2e = None
    if not args.no_e2e:
        hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
        ho = torch.empty_like(hq).pin_memory()
        inp_bytes = 3 * hq.numel() * hq.element_size()
        out_bytes = ho.numel() * ho.element_size()
        if world == 1:
            path = "tcb.carve_layer on pinned host Q/K/V: head-chunked H2D / mask+carve / D2H on 3 streams"

            def e2e_step():
                tcb.carve_layer(hq, hk, hv, layout, statics, params, out=ho)
        else:
            from paper_2505_16864_b200.ulysses import carve_layer_sp
            path = ("per rank: pinned host token shard -> H2D -> ulysses.carve_layer_sp (all-to-all, "
                    "build_block_mask + carve_attention on the head shard, all-to-all) -> D2H")

            def local_api(qh, kh, vh, lay, out):
                mask, _ = tcb.build_block_mask(qh, kh, lay, statics, params, need_relevance=False)
                tcb.carve_raw(qh, kh, vh, mask, lay, 0.0, out=out)

            def e2e_step():
                dq, dk, dv = (t.to(dev, non_blocking=True) for t in (hq, hk, hv))
                o_sh = carve_layer_sp(dq, dk, dv, layout, local_api, chunks=args.a2a_chunks)
                ho.copy_(o_sh, non_blocking=True)
                torch.cuda.current_stream().synchronize()

        e2e_step()
        barrier()
        n_e2e = max(2, min(args.steps, 5))
        a, b = ev(), ev()
        a.record()
        for _ in range(n_e2e):
            e2e_step()
        b.record()
        barrier()
        e2e_ms = a.elapsed_time(b) / n_e2e
        if world > 1:
            t = torch.tensor([e2e_ms], device=red_dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": inp_bytes * world,
               "d2h_bytes_per_step": out_bytes * world, "path": path}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_seconds)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "carve_traffic.json")
    if world == 1 and os.path.exists(tpath):  # the capture is of the 1-GPU C2 launch
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": round(ms_step, 4),
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (torch.randn Q/K/V, bf16), random-init; no checkpoint",
        "config": {"workload": WORKLOAD, "tokens": Np, "heads": H, "d": D, "block": M,
                   "k": K_RATE, "p": P_CUT, "kept_pairs": pairs,
                   "kept_fraction": round(pairs / (H * Mt * Mt), 4),
                   "parallelism": (f"ulysses-heads{world}-a2a{args.a2a_chunks}chunks-exchange-layout")
                   if world > 1 else "single",
                   "l2": "no flush: Q/K/V/O = 2.9 GB per layer > 126 MB L2"},
        "kept_block_tflops": round(carve_tflops, 1),
        "layer_tflops": round(flops / (ms_step * 1e-3) / 1e12, 1),
        "cuda_graph_ms_per_step": graph_ms,
        "kernels_ms": None if chunked else {
            "block_pool": round(float(k_pool), 4),
            "block_mask (scores + select + union, no R)": round(float(k_sel), 4),
            "carve_fwd": round(float(k_carve), 4)},
        "roofline": {"bound": "tensor", "kernel": "k_carve_tc<128>",
                     "achieved": round(carve_tflops, 1), "peak": tf_burst, "unit": "TFLOP/s",
                     "frac": round(carve_tflops / tf_burst, 4),
                     "peak_source": f"{peak_src} bf16_tflops (burst: the kernel runs at ~1.4-1.6 GHz, "
                                    "above the sustained GEMM's 1.32 GHz, so burst is the honest ceiling)",
                     "frac_of_sustained": round(carve_tflops / tf_sust, 4),
                     "traffic": traffic,
                     "algorithmic_flops_per_launch": flops_local,
                     "pool_hbm_gbs": None if chunked else round(2 * Hl * Np * D * 2 / (k_pool * 1e-3) / 1e9, 1),
                     "hbm_peak_gbs": hbm},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": 5 * args.steps * (args.a2a_chunks if chunked else 1),
        "launches_per_layer": "k_pool, k_scores_dmma, k_select (scores, p=0 fast path), k_select "
                              "(exact re-run of near-tie rows only), k_carve_tc",
        "clocks": clk.result,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------ CPU arm
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_module():
    """The unmodified reference package installed into baseline/_ref (pip --target, see
    DESIGN.md §7), or None when it is absent (then the oracle port stands in)."""
    if not os.path.isdir(os.path.join(REF_DIR, "tokencarve")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import tokencarve

    if not os.path.abspath(tokencarve.__file__).startswith(REF_DIR):
        return None
    return tokencarve


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuLayer:
    """The C2 layer on the host: the reference's own build_block_mask over all 24 heads
    (timed once) and its per-(head, q-block) carve body, timed on consecutive slices of the
    reference's job list (attention.py:236-239), so successive steps cover whole heads.

    Q/K/V are the same bf16-representable values the GPU arm computes on (default_rng(0)
    normals rounded to bf16, held as fp32 -- the reference's only precision)."""

    def __init__(self):
        from threadpoolctl import threadpool_limits

        self.tc = reference_module()
        self.kind = "reference" if self.tc is not None else "port"
        self.threads = len(os.sched_getaffinity(0))
        self._limits = threadpool_limits(limits=1, user_api="blas")  # workers x 1 BLAS thread
        rng = np.random.default_rng(0)
        import torch

        Np = math.ceil(DIMS[0] * DIMS[1] * DIMS[2] / M) * M + math.ceil(N_COND / M) * M
        shape = (H, Np, D)
        self.q, self.k, self.v = (
            torch.from_numpy(rng.standard_normal(shape, dtype=np.float32)).to(torch.bfloat16)
            .to(torch.float32).numpy() for _ in range(3))
        t0 = time.perf_counter()
        if self.tc is not None:
            tc = self.tc
            dims = tc.GridDims(*DIMS)
            self.layout = tc.build_layout(dims, M, N_COND)
            statics = tc.StaticMasks.build(self.layout, dims, tc.build_curve(dims))
            t0 = time.perf_counter()
            mask, _ = tc.build_block_mask(self.q, self.k, self.layout, statics,
                                          tc.SelectionParams(k=K_RATE, p=P_CUT))
            self.t_mask = time.perf_counter() - t0
            self.bits = mask.bits
            self.inputs = tc.AttentionInputs(q=self.q, k=self.k, v=self.v, layout=self.layout)
            from tokencarve.attention import _carve_rows

            self._rows = _carve_rows
            M_v, M_total = self.layout.M_v, self.layout.M_total
        else:
            import oracle

            self.L = oracle.layout_scalars(DIMS, M, N_COND)
            adja = oracle.adjacency(DIMS, oracle.curve_inverse(oracle.curve_forward(DIMS)), M,
                                    self.L["M_v"])
            t0 = time.perf_counter()
            self.bits, _ = oracle.block_mask(self.q, self.k, self.L, adja, K_RATE, P_CUT)
            self.t_mask = time.perf_counter() - t0
            M_v, M_total = self.L["M_v"], self.L["M_total"]
        self.out = np.zeros_like(self.q)
        row = self.bits.sum(axis=-1)
        self.jobs = [(h, b) for h in range(H) for b in range(M_total)]  # attention.py:236
        self.job_pairs = [int(row[h, b]) if b < M_v else M_total for h, b in self.jobs]
        self.total_pairs = int(sum(self.job_pairs))
        self.pos = 0
        self.covered = 0  # jobs timed so far (consecutive from job 0)

    def _run(self, jobs):
        from concurrent.futures import ThreadPoolExecutor

        if self.tc is not None:
            f = lambda hb: self._rows(self.inputs, self.bits, 0.0, *hb, self.out)  # noqa: E731
            with ThreadPoolExecutor(max_workers=self.threads) as pool:  # attention.py:237-239
                list(pool.map(f, jobs))
        else:
            import oracle

            oracle.carve(self.q, self.k, self.v, self.bits, self.L, 0.0, workers=self.threads,
                         items=jobs)

    def step(self, budget_s: float) -> float:
        """Carve the next jobs for about budget_s; returns the extrapolated ms per layer
        (measured s/pair x all kept pairs + the 24-head mask build)."""
        t, pairs = 0.0, 0
        chunk = 4 * self.threads
        while t < budget_s:
            if self.pos >= len(self.jobs):
                self.pos = 0
            sel = self.jobs[self.pos:self.pos + chunk]
            t0 = time.perf_counter()
            self._run(sel)
            t += time.perf_counter() - t0
            pairs += sum(self.job_pairs[self.pos:self.pos + len(sel)])
            self.pos += len(sel)
            self.covered = max(self.covered, self.pos)
        return (t / pairs * self.total_pairs + self.t_mask) * 1e3

    def describe(self) -> str:
        heads = min(H, self.covered // (len(self.jobs) // H))
        what = ("reference tokencarve 0.1.0 from baseline/_ref (unmodified; build_block_mask + "
                "attention._carve_rows, the body carve_attention maps over its ThreadPoolExecutor)"
                if self.tc is not None else "oracle port of the reference (baseline/_ref absent)")
        return (f"{what}, fp32, {self.threads} worker threads x 1 BLAS thread on {self.threads} "
                f"cores ({cpu_model()}): build_block_mask over all {H} heads once "
                f"({self.t_mask:.2f} s, added to every step) + carve of consecutive "
                f"(head, q-block) jobs, {self.covered} jobs timed = {heads} whole heads; "
                f"per-step value = measured s per kept pair x {self.total_pairs} kept pairs "
                f"(extrapolation factor {self.total_pairs / max(1, self._covered_pairs()):.2f}) "
                f"+ the mask build")

    def _covered_pairs(self) -> int:
        return sum(self.job_pairs[: self.covered])


def cpu_baseline(budget_s):
    cl = CpuLayer()
    ms = cl.step(budget_s)
    return {"value": round(ms, 1), "unit": "ms", "cores": cl.threads, "kind": cl.kind,
            "sample": cl.describe()}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cl = CpuLayer()
    # keep the whole run within a few minutes: ~200 s of carving over all steps
    budget = max(2.0, 200.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cl.step(budget)
    vals = [cl.step(budget) for _ in range(args.steps)]
    v = float(np.mean(vals))
    line = {"metric": METRIC, "value": round(v, 1), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 1),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (the reference's only precision; Q/K/V are the bf16-rounded values)",
            "data": "synthetic (numpy default_rng(0) normals rounded to bf16, held as fp32)",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "tokens": len(cl.q[0]), "heads": H, "d": D,
                       "block": M, "k": K_RATE, "p": P_CUT, "kept_pairs": cl.total_pairs},
            "cpu_baseline": {"value": round(v, 1), "unit": "ms", "cores": cl.threads,
                             "kind": cl.kind, "sample": cl.describe()},
            "e2e": {"value": round(v, 1), "unit": "ms", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--a2a-chunks", type=int, default=None,
                    help="N>1: pipeline the Ulysses all-to-all over this many head chunks "
                         "(default: 2 when a rank holds an even number >= 2 of heads)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

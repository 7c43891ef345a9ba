"""Benchmark of the DynSplit-KV decode hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Workload (config.workload): BASELINE.json config 3's per-GPU shard -- a
Llama-3-8B-shaped decode step (32 layers, 32 Q / 8 KV heads, d = 128, bf16 KV)
at 128K context, token budget 4096, `--batch-per-gpu` sequences per GPU
(default 1, so N = 8 is config 3's batch 8 sharded by batch).  A step = one
decode token through all 32 layers: per layer dynsplit_decode_layer = a5 block
scoring + a6 budgeted selection + a7/a8 split-K sparse attention with LSE
merge, all in libdynsplit.so kernels, replayed as one CUDA graph.  Sequences are independent
(no data-path collective); scaling is weak (fixed work per GPU).

value = aggregate algorithmic HBM bytes per step (digests + GQA-union of the
selected K/V rows + block starts + q + o/lse) over all
ranks / max-over-ranks step time, in GB/s.  ms_per_step is the decode step
latency.  The per-layer working set (~65 MiB x 32 layers ~ 2 GiB per step) is
far larger than the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse decode-attn µs/step & HBM GB/s vs peak at 128K ctx, 1/2/4/8 B200"
WORKLOAD = "C3 per-GPU shard: Llama-3-8B decode (32 layers, 32Q/8KV, d=128, bf16) at 128K ctx, budget 4K"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch-per-gpu", type=int, default=1)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--budget", type=int, default=4096)
    ap.add_argument("--rho", type=float, default=0.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--cpu-sample-heads", type=int, default=32)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/traffic.json), or None."""
    try:
        j = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return float(j[kernel]["dram_bytes_per_launch"])
    except Exception:
        return None


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every
    ~2 ms while the timed region runs (nvidia-smi as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.sm = []
        self.mask = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            p = self._nvml
            self.sm.append(float(p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)))
            self.mask |= int(p.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        self.sm.append(float(out[0]))
        self.max_mhz = float(out[1])
        self.mask |= int(out[2], 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.sm)}


# ---------------------------------------------------------------------------
# oracle (CPU) timing: the cpu_baseline leg and the --impl reference arm
# ---------------------------------------------------------------------------
def oracle_layer_bytes(q, K, starts, budget, Hkv, g, e=2):
    """Algorithmic bytes of one decode step of one layer of one sequence
    (same accounting as the GPU line), from the oracle's own selection."""
    from oracle import dynsplit_oracle as O
    nb = len(starts) - 1
    res_tokens = []
    kmax, kmin = O.digests(K, starts)
    for h in range(q.shape[0]):
        sc = O.block_scores(q[h], kmax[h // g], kmin[h // g])
        res_tokens.append(set(O.select_tokens(sc, starts, budget).tolist()))
    union = sum(len(set().union(*res_tokens[hk * g:(hk + 1) * g])) for hk in range(Hkv))
    d = q.shape[1]
    return nb * Hkv * 2 * d * e + union * 2 * d * e + 2 * (nb + 1) * 4 + q.size * e + q.shape[0] * (d + 1) * 4


def time_oracle(q, K, V, starts, budget, heads):
    """Oracle decode step over the sampled heads; returns seconds."""
    from oracle import dynsplit_oracle as O
    t0 = time.perf_counter()
    O.decode_step(q[:heads], K, V, starts, budget)
    return time.perf_counter() - t0


def host_layer(seed, S, Hq, Hkv, d, rho):
    from synth import generators as G
    return G.decode_qkv(seed, S, Hq, Hkv, d, rho=rho)


def cpu_threads_limit():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import dynsplit_oracle as O
    from synth import generators as G
    S, Hq, Hkv, d = args.seq, args.hq, args.hkv, 128
    g = Hq // Hkv
    toks = G.tokens(args.seed, S)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
    q, K, V = host_layer(args.seed, S, Hq, Hkv, d, args.rho)
    heads = min(args.cpu_sample_heads, Hq)
    frac = heads / Hq
    layer_bytes = oracle_layer_bytes(q, K, starts, args.budget, Hkv, g)
    times = []
    with cpu_threads_limit():
        for i in range(args.warmup + args.steps):
            dt = time_oracle(q, K, V, starts, args.budget, heads)
            if i >= args.warmup:
                times.append(dt)
    sec = float(np.mean(times))
    # one oracle step = `heads` of the 32 heads of one layer of one sequence;
    # scaled to the metric: bytes that fraction of a layer touches per second
    gbs = layer_bytes * frac / sec / 1e9
    step_ms = sec / frac * args.layers * args.batch_per_gpu * 1e3
    sample = f"oracle decode step, {heads}/{Hq} heads of 1 layer of 1 seq at S={S}, budget {args.budget}"
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "seq_len": S, "layers": args.layers,
                       "batch_per_gpu": args.batch_per_gpu, "budget": args.budget},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# prefill context line: config 5 block construction, one scored layer
# ---------------------------------------------------------------------------
def prefill_c5(args, D, G, cfg, ids, dev, cur):
    """BASELINE.json config 5 (Llama-3-8B shape, 64K, batch 4): rows a1-a4 of
    block construction, each stage timed with CUDA events after a warm-up
    (outputs preallocated).  Context for the decode headline, not part of it."""
    import torch
    S_pf, B_pf, Hq, Hkv, d = 65536, 4, args.hq, args.hkv, 128
    gpf = torch.Generator(device=dev)
    gpf.manual_seed(args.seed + 17)
    toks = torch.from_numpy(np.stack([G.tokens(args.seed * 31 + b, S_pf) for b in range(B_pf)])).to(dev)
    Qs = torch.randn(1, B_pf, S_pf, Hq, d, generator=gpf, device=dev).to(torch.bfloat16)
    Ks = torch.randn(1, B_pf, S_pf, Hkv, d, generator=gpf, device=dev).to(torch.bfloat16)
    K = torch.randn(B_pf, S_pf, Hkv, d, generator=gpf, device=dev).to(torch.bfloat16)
    V = torch.randn(B_pf, S_pf, Hkv, d, generator=gpf, device=dev).to(torch.bfloat16)

    def timed(fn, reps):
        # median over reps of per-call event pairs (a one-off host-side
        # allocation stall between the events would otherwise count as GPU time)
        out = fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cur)
            out = fn()
            b.record(cur)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts)), out

    t1, s = timed(lambda: D.score_delimiters(toks, ids, Qs, Ks, cfg), 3)
    t2, w10 = timed(lambda: D.weight_table(toks, ids, s), 5)
    t3, (bs, nb) = timed(lambda: D.segment(toks, ids, w10, cfg), 5)
    t4a, (pf, _, _, _) = timed(lambda: D.map_pages(bs, nb, S_pf, cfg), 5)
    kvd = D.repack_digest(K, V, bs, nb, pf, cfg)
    t4b, _ = timed(lambda: D.repack_digest(K, V, bs, nb, pf, cfg, out=kvd), 5)
    rows = np.arange(S_pf, dtype=np.float64) + 1
    flop = 2.0 * d * Hq * rows.sum() * B_pf            # causal Q.K^T of every query row
    exps = Hq * rows.sum() * B_pf
    a4_bytes = 2 * 2 * B_pf * S_pf * Hkv * d * 2 + int(nb.sum()) * Hkv * 2 * d * 2   # K, V read + written, digests
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        tf_peak, hbm_peak, src = float(pk["bf16_tflops_sustained"]), float(pk["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        tf_peak, hbm_peak, src = 1395.5, 6650.0, "fallback (B200_PROFILING.md)"
    del Qs, Ks, K, V, kvd
    return {"config": f"C5: block construction, Llama-3-8B shape ({Hq}Q/{Hkv}KV, d=128, bf16), "
                      f"S={S_pf}, batch {B_pf}, 1 scored layer",
            "ms_total": t1 + (t2 + t3 + t4a + t4b),
            "a1_ms": t1, "a1_tflops": flop / (t1 * 1e-3) / 1e12, "a1_tflops_frac": flop / (t1 * 1e-3) / 1e12 / tf_peak,
            "a1_exp_per_s": exps / (t1 * 1e-3),
            "a2_us": t2 * 1e3, "a3_us": t3 * 1e3, "a4_map_us": t4a * 1e3, "a4_repack_us": t4b * 1e3,
            "a4_GBs": a4_bytes / (t4b * 1e-3) / 1e9, "a4_frac": a4_bytes / (t4b * 1e-3) / 1e9 / hbm_peak,
            "blocks_per_seq": int(nb[0]),
            "note": "a1 k_lse_band_tc (tcgen05 UMMA into TMEM + MUFU ex2), peaks from " + src}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    from paper_2602_03184_b200 import dynsplit as D
    from synth import generators as G

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    D.lib()

    B, S, Hq, Hkv, d, L = args.batch_per_gpu, args.seq, args.hq, args.hkv, 128, args.layers
    g = Hq // Hkv
    budget = args.budget
    cfg = D.default_config()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000003 * (args.seed + 1) + rank)

    # ---- prefill (untimed setup): tokens -> static-T7 DD-Select plan, pages, digests
    toks = torch.from_numpy(np.stack([G.tokens(args.seed * 7919 + rank * B + b, S) for b in range(B)])).to(dev)
    ids = torch.from_numpy(G.T7_IDS).to(dev)
    layers, qs = [], []
    host_keep = None
    for l in range(L):
        q, K, V = G.torch_decode_layer(gen, S, Hq, Hkv, d, B, dev, rho=args.rho)
        layers.append(D.build_blocks(toks, ids, K, V, cfg, static_w10=G.T7_W10, Hq=Hq))
        qs.append(q.contiguous())
        if l == 0 and rank == 0 and not args.no_cpu_baseline:
            host_keep = (q[0].float().cpu().numpy(), K[0].float().cpu().numpy(), V[0].float().cpu().numpy())
        del K, V
    torch.cuda.synchronize()

    # ---- per-layer preallocated outputs; shared workspaces / worklist
    shape = D.make_shape(B, S, Hq, Hkv, d)
    sel_out = [D._sel_outputs(shape, cfg, budget, dev, want_blocks=False) for _ in range(L)]
    attn_out = [(torch.empty(B, Hq, d, device=dev), torch.empty(B, Hq, device=dev)) for _ in range(L)]
    ws_sel = D.workspace(D.workspace_bytes(D.OP_SELECT, shape, cfg, budget), dev, "select")
    ws_dec = D.workspace(D.workspace_bytes(D.OP_DECODE_ATTN, shape, cfg), dev, "decode")

    def sel_layer(l):
        sb, ns, mg, kp, wl = sel_out[l]
        return D.select(qs[l], layers[l], budget, out=(sb, ns, mg, kp, wl, None), ws=ws_sel)

    def attn_layer(l):
        return D.decode_attn(qs[l], layers[l], sel_out[l][4], out=attn_out[l], ws=ws_dec)

    ws_step = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "layer_step")

    def step():
        # the public per-layer call (a5 -> a6 -> a7+a8, PDL-ordered)
        for l in range(L):
            _, ns, mg, kp, wl = sel_out[l]
            D.decode_layer(qs[l], layers[l], budget, out=(ns, mg, kp, wl, attn_out[l][0], attn_out[l][1]),
                           ws=ws_step)

    def dense_step():
        for l in range(L):
            D.decode_attn(qs[l], layers[l], None, out=attn_out[l], ws=ws_dec)

    # eager warm-up call (sets kernel attributes before capture), metrics
    step()
    torch.cuda.synchronize()
    e = 2
    nblk = [int(x) for x in layers[0].n_blocks.cpu()]
    union_rows = 0
    for l in range(L):
        _, streamed = D.worklist_rows(sel_out[l][4], shape, g)
        union_rows += int(streamed.sum())
    n_entries_total = 0
    digest_bytes = L * sum(nblk) * Hkv * 2 * d * e
    kv_bytes = union_rows * 2 * d * e
    small = L * (2 * sum(n + 1 for n in nblk) * 4 + B * Hq * d * e + B * Hq * (d + 1) * 4)
    step_bytes = digest_bytes + kv_bytes + small
    attn_bytes_per_launch = (kv_bytes + L * (B * Hq * d * e + B * Hq * (d + 1) * 4)) / L
    score_bytes_per_launch = digest_bytes / L + B * Hq * d * e

    # ---- CUDA graphs: whole step; per-layer select / attn (kernel timing)
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream(dev).wait_stream(s)
    g_step = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_step):
        step()
    # per-kernel-group timing: all L layers' a5+a6 (resp. a7+a8) launches in one
    # graph, back to back as in the step (PDL-chained), averaged per launch
    g_sel_all, g_attn_all = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_sel_all):
        for l in range(L):
            sel_layer(l)
    # a5 alone (block scores into the select workspace), for the a5 / a6 split
    mb_ = D.max_blocks(S, cfg)
    score_buf = torch.empty(B, Hq, mb_, dtype=torch.float32, device=dev)
    g_score_all = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_score_all):
        for l in range(L):
            D.score_blocks(qs[l], layers[l], out=score_buf)
    with torch.cuda.graph(g_attn_all):
        for l in range(L):
            attn_layer(l)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        g_step.replay()
    barrier()

    # ---- timed region 1: whole-step graph
    cur = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    # clocks are sampled over timed regions 1 and 2 (the step graph, then the
    # per-kernel-group graphs): region 1 alone is only ~50 ms at the defaults
    clk = ClockSampler(local)
    clk.__enter__()
    barrier()
    ev0.record(cur)
    for i in range(args.steps):
        step_evs[i].record(cur)
        g_step.replay()
    step_evs[-1].record(cur)
    ev1.record(cur)
    barrier()
    step_ms = ev0.elapsed_time(ev1) / args.steps
    per_step = np.array([step_evs[i].elapsed_time(step_evs[i + 1]) for i in range(args.steps)])

    # ---- timed region 2: the step's kernel groups, each as an L-layer graph
    barrier()
    t0, t1, t2, t3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    t0.record(cur)
    for _ in range(args.steps):
        g_sel_all.replay()
    t1.record(cur)
    for _ in range(args.steps):
        g_attn_all.replay()
    t2.record(cur)
    for _ in range(args.steps):
        g_score_all.replay()
    t3.record(cur)
    barrier()
    clk.__exit__(None, None, None)
    sel_ms = t0.elapsed_time(t1) / (args.steps * L)
    attn_ms = t1.elapsed_time(t2) / (args.steps * L)
    score_ms = t2.elapsed_time(t3) / (args.steps * L)
    split_step_ms = t0.elapsed_time(t2) / args.steps

    # ---- e2e: the step's inputs from pinned HOST memory (every layer's q, one
    #      H2D copy), the public per-layer call dynsplit_decode_layer, and the
    #      step's result (every layer's o and lse) read back to pinned host
    #      memory (one D2H copy) and synchronised on, every step
    q_all_h = torch.stack([q.cpu() for q in qs]).pin_memory()            # [L, B, Hq, d] bf16
    # every layer's o and lse in one buffer, read back with one D2H copy
    res_h = torch.empty(L * B * Hq * (d + 1)).pin_memory()
    q_all_d = torch.empty(q_all_h.shape, dtype=q_all_h.dtype, device=dev)
    res_d = torch.empty(L * B * Hq * (d + 1), device=dev)
    o_all_d = res_d[: L * B * Hq * d].view(L, B, Hq, d)
    l_all_d = res_d[L * B * Hq * d:].view(L, B, Hq)
    ws_layer = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "layer_e2e")
    sel_e2e = D._sel_outputs(shape, cfg, budget, dev, want_blocks=False)

    def host_step():
        q_all_d.copy_(q_all_h, non_blocking=True)
        for l in range(L):
            _, ns, mg, kp, wl = sel_e2e
            D.decode_layer(q_all_d[l], layers[l], budget, out=(ns, mg, kp, wl, o_all_d[l], l_all_d[l]),
                           ws=ws_layer)
        res_h.copy_(res_d, non_blocking=True)

    host_step()
    torch.cuda.synchronize()
    g_host = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_host):
        host_step()
    for _ in range(args.warmup):
        g_host.replay()
    barrier()
    ev0.record(cur)
    for _ in range(args.steps):
        g_host.replay()
        cur.synchronize()                     # the step's result is read on the host
    ev1.record(cur)
    barrier()
    e2e_ms = ev0.elapsed_time(ev1) / args.steps
    h2d = q_all_h.numel() * q_all_h.element_size()
    d2h = res_h.numel() * 4

    # ---- prefill row a1 (context, not the headline): Alg. 1 delimiter scoring
    #      of one sequence-layer at S_pf (C5 shape: 32Q/8KV, bf16), one launch pair
    prefill = None
    if rank == 0 and not args.no_prefill:
        prefill = prefill_c5(args, D, G, cfg, ids, dev, cur)

    # ---- dense baseline (row a9): every page, every head
    dense_ms = None
    if not args.no_dense:
        g_dense = torch.cuda.CUDAGraph()
        dense_step()
        torch.cuda.synchronize()
        with torch.cuda.graph(g_dense):
            dense_step()
        g_dense.replay()
        barrier()
        nd = max(2, min(args.steps, 5))
        ev0.record(cur)
        for _ in range(nd):
            g_dense.replay()
        ev1.record(cur)
        barrier()
        dense_ms = ev0.elapsed_time(ev1) / nd

    # ---- max over ranks
    vals = torch.tensor([step_ms, attn_ms, sel_ms, e2e_ms, split_step_ms, dense_ms or 0.0, score_ms],
                        dtype=torch.float64, device=dev)
    tot_bytes = torch.tensor([float(step_bytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_bytes, op=dist.ReduceOp.SUM)
    step_ms, attn_ms, sel_ms, e2e_ms, split_step_ms, dense_ms_v, score_ms = vals.tolist()
    all_bytes = tot_bytes.item()

    cpu = None
    if rank == 0 and host_keep is not None:
        from oracle import dynsplit_oracle as O
        qh, Kh, Vh = host_keep
        starts = O.segment(G.tokens(args.seed * 7919 + 0, S), G.T7_IDS, G.T7_W10, 32, 14)
        heads = min(args.cpu_sample_heads, Hq)
        lb = oracle_layer_bytes(qh, Kh, starts, budget, Hkv, g)
        ts = []
        with cpu_threads_limit():
            t_start = time.perf_counter()
            while not ts or (time.perf_counter() - t_start < args.cpu_seconds and len(ts) < 50):
                ts.append(time_oracle(qh, Kh, Vh, starts, budget, heads))
        sec = float(np.mean(ts))
        cpu = {"value": lb * heads / Hq / sec / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"{len(ts)} oracle decode steps of layer 0, sequence 0 ({heads}/{Hq} heads) "
                         f"at S={S}, budget {budget}; mean {sec:.2f} s each, "
                         f"{sum(ts):.1f} s total, 1 thread"}

    if rank == 0:
        peak, peak_src = measured_peak_hbm()
        achieved = attn_bytes_per_launch / (attn_ms * 1e-3) / 1e9
        line = {
            "metric": METRIC,
            "value": all_bytes / (step_ms * 1e-3) / 1e9,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch_per_gpu": B, "global_batch": B * world,
                       "seq_len": S, "layers": L, "heads_q": Hq, "heads_kv": Hkv, "head_dim": d,
                       "budget": budget, "rho": args.rho, "C": cfg.C, "delta": cfg.delta,
                       "page_size": cfg.page_size, "parallelism": f"batch-shard x{world}",
                       "l2": "no flush: ~%.0f MiB touched per step >> 126 MB L2" % (step_bytes / 2**20)},
            "us_per_step": step_ms * 1e3,
            "step_ms_p10_p50_p90": [float(np.percentile(per_step, p)) for p in (10, 50, 90)],
            "us_per_layer": step_ms * 1e3 / L,
            "bytes_per_step": step_bytes,
            "union_factor": union_rows / (L * B * Hkv * budget),
            "roofline": {"bound": "hbm", "kernel": "k_decode_attn (a7+a8)", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": ncu_traffic("k_decode_attn"),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": attn_bytes_per_launch,
                         "avg_launch_us": attn_ms * 1e3,
                         "timing": "CUDA events around an L-layer graph of the kernel's launches (back to back, "
                                   "PDL-chained), per launch",
                         "select_us_per_layer": sel_ms * 1e3,
                         "score_us_per_layer": score_ms * 1e3,
                         "score_frac_of_peak": score_bytes_per_launch / (score_ms * 1e-3) / 1e9 / peak,
                         "select_bytes_per_launch": score_bytes_per_launch,
                         "step_frac_of_peak": (step_bytes / (step_ms * 1e-3) / 1e9) / peak},
            "e2e": {"value": all_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
            "gpu_launches": 3 * L * args.steps,   # k_score_blocks_tc, k_select_reg, k_decode_attn per layer
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        if prefill:
            line["prefill"] = prefill
        if dense_ms:
            dense_bytes = L * B * Hkv * S * 2 * d * e
            line["dense"] = {"ms_per_step": dense_ms_v, "GB_s": dense_bytes / (dense_ms_v * 1e-3) / 1e9,
                             "sparse_speedup": dense_ms_v / step_ms}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

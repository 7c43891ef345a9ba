"""Benchmark of the DynSplit-KV decode hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode batch|seqsplit]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

--mode batch (default; the headline).  Workload (config.workload): BASELINE.json
config 3's per-GPU shard -- a Llama-3-8B-shaped decode step (32 layers, 32 Q /
8 KV heads, d = 128, bf16 KV) at 128K context, token budget 4096,
`--batch-per-gpu` sequences per GPU (default 1, so N = 8 is config 3's batch 8
sharded by batch).  A step = one decode token through all 32 layers: per
layer one dynsplit_decode_layer call = one k_decode_fused launch (a5 block
scoring + a6 budgeted selection + a7/a8 split-K sparse attention with the LSE
merge), replayed as one CUDA graph.  Sequences are independent (no data-path
collective); scaling is weak (fixed work per GPU).  At N = 1 the line also
carries two more configurations of the metric, each with its roofline, e2e
and dense baseline: "c3_b8" (config 3 unsharded: all 8 sequences on one GPU)
and "c4" (config 4 on one GPU: Llama2-13B shape, 40 MHA heads, 40 layers).

--mode seqsplit.  Config 4 (Llama2-13B: 40 layers, 40 MHA heads, 128K,
budget 4096) sequence-split across the N ranks (parallel.SeqSplitDecoder:
local a5 -> NCCL all-gather of the block scores -> global a6 -> local a7 ->
all-gather of (o, lse) -> rank-ordered a8 merge); strong scaling.

value = aggregate algorithmic HBM bytes per step (digests + GQA-union of the
selected K/V rows + block starts + q + o/lse) over all
ranks / max-over-ranks step time, in GB/s; ms_per_step is the decode-step
latency.  The per-layer working set (~65 MiB x 32 layers ~ 2 GiB per step) is
far larger than the 126 MB L2, so no flush is needed between steps; blocks
that cycle fewer distinct layer caches than layers still stream every layer's
bytes from HBM (each cache is >> L2) and say so in their config.
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
WORKLOAD_C4 = "C4: Llama2-13B decode (40 layers, 40 MHA heads, d=128, bf16) at 128K ctx, budget 4K, sequence split"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="batch", choices=["batch", "seqsplit"])
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
    ap.add_argument("--no-extra", action="store_true", help="skip the c3_b8 / c4 blocks")
    ap.add_argument("--no-e2e-model", action="store_true", help="skip the NEXT-4 decoder block")
    ap.add_argument("--no-offload", action="store_true", help="skip the NEXT-3 offloaded-KV block")
    ap.add_argument("--only-offload", action="store_true", help="run only the NEXT-3 block (development)")
    ap.add_argument("--cpu-sample-heads", type=int, default=32)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


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


_POOL_ARGS = None  # (q, K, V, starts, budget) shared with forked workers


def _oracle_heads(hs):
    from oracle import dynsplit_oracle as O
    q, K, V, starts, budget = _POOL_ARGS
    g = q.shape[0] // K.shape[1]
    # the oracle's decode step over a contiguous group of query heads (whole KV groups)
    return O.decode_step(q[hs[0]:hs[1]], K[:, hs[0] // g: (hs[1] - 1) // g + 1], V[:, hs[0] // g: (hs[1] - 1) // g + 1],
                         starts, budget)["lse"].shape


def time_oracle(q, K, V, starts, budget, heads, workers=1):
    """Oracle decode step over the first `heads` query heads; returns seconds.
    workers > 1: whole KV groups of heads spread over forked processes."""
    global _POOL_ARGS
    from oracle import dynsplit_oracle as O
    if workers <= 1:
        t0 = time.perf_counter()
        O.decode_step(q[:heads], K, V, starts, budget)
        return time.perf_counter() - t0
    import multiprocessing as mp
    g = q.shape[0] // K.shape[1]
    groups = heads // g
    n = max(1, min(workers, groups))
    cuts = [round(i * groups / n) * g for i in range(n + 1)]
    _POOL_ARGS = (q, K, V, starts, budget)
    ctx = mp.get_context("fork")
    with ctx.Pool(n) as pool:
        t0 = time.perf_counter()
        pool.map(_oracle_heads, [(cuts[i], cuts[i + 1]) for i in range(n) if cuts[i + 1] > cuts[i]])
        dt = time.perf_counter() - t0
    return dt


def cpu_threads_limit():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def host_layer(seed, S, Hq, Hkv, d, rho):
    from synth import generators as G
    return G.decode_qkv(seed, S, Hq, Hkv, d, rho=rho)


def run_reference(args, world, rank):
    """The reference arm: the fp64 oracle (no reference implementation exists,
    the reference is a paper) on the host cores, one thread, on a bounded
    sample of the workload: each timed step is the oracle's decode step of
    `--cpu-sample-heads` query heads of ONE layer of one sequence.  The line's
    ms_per_step is that sample step as timed (steps x ms_per_step is the wall
    time of the timed region); the full-step time it extrapolates to (x layers
    x heads) is reported beside it, marked as such."""
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
    gbs = layer_bytes * frac / sec / 1e9
    sample = (f"oracle decode step, {heads}/{Hq} heads of 1 of {args.layers} layers of 1 sequence at S={S}, "
              f"budget {args.budget}, 1 thread")
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "seq_len": S, "layers": args.layers,
                       "batch_per_gpu": args.batch_per_gpu, "budget": args.budget},
            "sample_step": {"layers": 1, "heads": heads, "sequences": 1,
                            "extrapolated_full_step_ms": sec / frac * args.layers * args.batch_per_gpu * 1e3,
                            "note": "ms_per_step is the timed sample step; the full step is extrapolated"},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": cpu_model()},
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
    flop = 2.0 * d * Hq * rows.sum() * B_pf            # executed: causal Q.K^T of every query row
    exps = Hq * rows.sum() * B_pf
    # algorithmic work: only the rows q in the union of the
    # candidates' future windows F_i = {i+1 .. min(i+W, S-1)} are needed:
    # 2 d Hq sum_{q in UF} (q+1) FLOP and Hq sum (q+1) exps, plus the band
    # recompute 2 d Hq (W+R) |UF|
    W, R = cfg.W, cfg.R
    dset = np.isin(toks.cpu().numpy(), G.T7_IDS)
    need = np.zeros_like(dset)
    for w in range(1, W + 1):
        need[:, w:] |= dset[:, :-w]
    need[:, 0] = False
    n_need = int(need.sum())
    q_need = (np.nonzero(need)[1].astype(np.float64) + 1).sum()
    flop_alg = 2.0 * d * Hq * q_need + 2.0 * d * Hq * (W + R) * n_need
    exps_alg = Hq * q_need
    try:
        sm_mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        sm_mhz = 1965.0
    import torch as _t
    n_sm = _t.cuda.get_device_properties(dev).multi_processor_count
    mufu_peak = 16.0 * n_sm * sm_mhz * 1e6               # ex2 per second: 16 / clk / SM (B200_PROFILING)
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
            "a1_roofline": {"bound": "alu", "unit": "exp/s (MUFU ex2)", "peak": mufu_peak,
                            "achieved_executed": exps / (t1 * 1e-3),
                            "frac_executed": exps / (t1 * 1e-3) / mufu_peak,
                            "achieved_algorithmic": exps_alg / (t1 * 1e-3),
                            "frac_algorithmic": exps_alg / (t1 * 1e-3) / mufu_peak,
                            "rows_needed_frac": n_need / (B_pf * S_pf),
                            "algorithmic_tflops": flop_alg / (t1 * 1e-3) / 1e12,
                            "peak_note": f"16 ex2/clk/SM x {n_sm} SMs x {sm_mhz:.0f} MHz; the kernel computes every "
                                         f"causal row (no row compaction), so executed > algorithmic"},
            "a2_us": t2 * 1e3, "a3_us": t3 * 1e3, "a4_map_us": t4a * 1e3, "a4_repack_us": t4b * 1e3,
            "a4_GBs": a4_bytes / (t4b * 1e-3) / 1e9, "a4_frac": a4_bytes / (t4b * 1e-3) / 1e9 / hbm_peak,
            "blocks_per_seq": int(nb[0]),
            "note": "a1 k_lse_band_tc (tcgen05 UMMA into TMEM + MUFU ex2), peaks from " + src}


# ---------------------------------------------------------------------------
# GPU arm: one decode workload (B sequences, L layers over Ld distinct caches)
# ---------------------------------------------------------------------------
class Workload:
    """Synthetic decode workload: B sequences of S tokens, the static-T7
    DD-Select plan, Ld distinct layer caches (pages sized tightly to the
    plan's page count), one query per layer cache."""

    def __init__(self, D, G, B, S, Hq, Hkv, Ld, rho, seed, dev, tok_seed0):
        import torch
        self.D, self.B, self.S, self.Hq, self.Hkv, self.Ld = D, B, S, Hq, Hkv, Ld
        d = 128
        self.d = d
        ids = torch.from_numpy(G.T7_IDS).to(dev)
        self.toks = torch.from_numpy(np.stack([G.tokens(tok_seed0 + b, S) for b in range(B)])).to(dev)
        cfg0 = D.default_config()
        plan = D.build_blocks(self.toks, ids, None, None, cfg0, static_w10=G.T7_W10, Hq=Hq, Hkv=Hkv)
        cap = int(plan.n_pages.max().item()) + 8                     # setup-time read of the plan
        self.cfg = D.default_config(page_cap=cap)
        self.nblk = [int(x) for x in plan.n_blocks.cpu()]
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.layers, self.qs = [], []
        self.host_keep = None
        for l in range(Ld):
            q, K, V = G.torch_decode_layer(gen, S, Hq, Hkv, d, B, dev, rho=rho)
            self.layers.append(D.build_blocks(self.toks, ids, K, V, self.cfg, static_w10=G.T7_W10, Hq=Hq))
            self.qs.append(q.contiguous())
            if l == 0:
                self.K0 = K[0].float().cpu().numpy()
                self.V0 = V[0].float().cpu().numpy()
                self.q0 = q[0].float().cpu().numpy()
            del K, V
        torch.cuda.synchronize()
        self.shape = D.make_shape(B, S, Hq, Hkv, d)


def time_graph(torch, fn, steps, warmup, cur, dev, world, barrier):
    """Capture fn() (one step) in a CUDA graph, replay `warmup` times, then time
    `steps` replays with events around each; returns (mean ms, per-step ms)."""
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream(dev).wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(warmup):
        g.replay()
    barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    for i in range(steps):
        evs[i].record(cur)
        g.replay()
    evs[-1].record(cur)
    barrier()
    per = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(steps)])
    return float(evs[0].elapsed_time(evs[-1]) / steps), per, g


def decode_block(args, torch, D, wl: Workload, L, budget, dev, cur, world, barrier, peak, with_e2e=True,
                 with_dense=True, with_three_kernel=False):
    """Time one decode workload: the step graph (L dynsplit_decode_layer calls
    = L k_decode_fused launches), its algorithmic bytes, the fused kernel's
    roofline, e2e through dynsplit_decode_step_host, the dense baseline."""
    B, Hq, Hkv, d = wl.B, wl.Hq, wl.Hkv, wl.d
    g = Hq // Hkv
    shape, cfg = wl.shape, wl.cfg
    Ld = wl.Ld
    outs = [(torch.empty(B, Hq, d, device=dev), torch.empty(B, Hq, device=dev)) for _ in range(L)]
    sel = [D._sel_outputs(shape, cfg, budget, dev, want_blocks=False) for _ in range(Ld)]
    ws = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "layer_step")

    def step():
        for l in range(L):
            j = l % Ld
            _, ns, mg, kp, w = sel[j]
            D.decode_layer(wl.qs[j], wl.layers[j], budget, out=(ns, mg, kp, w, outs[l][0], outs[l][1]), ws=ws)

    lib = D.lib()
    lib.dynsplit_debug_fused_launches.restype = __import__("ctypes").c_longlong
    n0 = lib.dynsplit_debug_fused_launches()
    step()
    torch.cuda.synchronize()
    fused_per_step = lib.dynsplit_debug_fused_launches() - n0
    # algorithmic bytes (digests + union rows + block starts + q + o/lse) from the worklists
    union_rows = []
    for j in range(Ld):
        _, streamed = D.worklist_rows(sel[j][4], shape, g)
        union_rows.append(int(streamed.sum()))
    e = 2
    per_layer = [sum(wl.nblk) * Hkv * 2 * d * e + union_rows[l % Ld] * 2 * d * e
                 + 2 * sum(n + 1 for n in wl.nblk) * 4 + B * Hq * d * e + B * Hq * (d + 1) * 4 for l in range(L)]
    step_bytes = float(sum(per_layer))
    ms, per, gstep = time_graph(torch, step, args.steps, args.warmup, cur, dev, world, barrier)
    res = {"ms_per_step": ms, "us_per_layer": ms * 1e3 / L, "bytes_per_step": step_bytes,
           "GB_s": step_bytes / (ms * 1e-3) / 1e9,
           "step_ms_p10_p50_p90": [float(np.percentile(per, p)) for p in (10, 50, 90)],
           "union_factor": sum(union_rows[l % Ld] for l in range(L)) / (L * B * Hkv * budget),
           "fused_launches_per_step": fused_per_step}
    # the dominant (only) kernel: k_decode_fused, one launch per layer
    kname = ("k_decode_fused (a5+a6+a7+a8)" if fused_per_step == L else
             "three kernels per layer: k_score_blocks_tc -> k_select_reg -> k_decode_attn (the fused layer "
             "declined this shape)")
    res["roofline"] = {"bound": "hbm", "kernel": kname,
                       "achieved": step_bytes / L / (ms * 1e-3 / L) / 1e9, "peak": peak[0], "unit": "GB/s",
                       "frac": step_bytes / (ms * 1e-3) / 1e9 / peak[0],
                       "traffic": ncu_traffic("k_decode_fused"), "peak_source": peak[1],
                       "algorithmic_bytes_per_launch": step_bytes / L, "avg_launch_us": ms * 1e3 / L,
                       "timing": "CUDA events around the step graph of L back-to-back (PDL-chained) launches, "
                                 "per launch"}
    if with_three_kernel:
        # context: the same step through the three-kernel path (a5 -> a6 -> a7), and
        # k_decode_attn alone (its old roofline)
        lib.dynsplit_debug_fused(0)
        try:
            ms3, _, _ = time_graph(torch, step, args.steps, args.warmup, cur, dev, world, barrier)
            wsd = D.workspace(D.workspace_bytes(D.OP_DECODE_ATTN, shape, cfg), dev, "decode")

            def attn_only():
                for l in range(L):
                    j = l % Ld
                    D.decode_attn(wl.qs[j], wl.layers[j], sel[j][4], out=outs[l], ws=wsd)
            msa, _, _ = time_graph(torch, attn_only, args.steps, args.warmup, cur, dev, world, barrier)
        finally:
            lib.dynsplit_debug_fused(1)
        attn_bytes = sum(union_rows[l % Ld] * 2 * d * e + B * Hq * d * e + B * Hq * (d + 1) * 4
                         for l in range(L)) / L
        res["three_kernel_path"] = {"ms_per_step": ms3, "k_decode_attn_us": msa * 1e3 / L,
                                    "k_decode_attn_frac": attn_bytes / (msa * 1e-3 / L) / 1e9 / peak[0],
                                    "note": "k_score_blocks_tc -> k_select_reg -> k_decode_attn per layer "
                                            "(DYNSPLIT_NO_FUSED), context"}
    if with_e2e:
        # e2e through the exported whole-step host-buffer call
        # dynsplit_decode_step_host_layers: every step ONE copy of every
        # layer's q from pinned host memory, the L decode layers, ONE copy
        # each of every layer's o and lse back to pinned host memory; the host
        # reads the step's result (synchronise)
        q_h = torch.stack([wl.qs[l % Ld].cpu() for l in range(L)]).pin_memory()
        o_h = torch.empty(L, B, Hq, d).pin_memory()
        l_h = torch.empty(L, B, Hq).pin_memory()
        lays = [wl.layers[l % Ld] for l in range(L)]
        wsh = D.workspace(D.step_host_layers_workspace_bytes(shape, cfg, budget, L), dev, "step_host_layers")
        wlh = D._sel_outputs(shape, cfg, budget, dev, want_blocks=False)[4]

        def host_step():
            D.decode_step_host_layers(q_h, lays, budget, o_h, l_h, wlh, wsh)

        for _ in range(args.warmup):
            host_step()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(cur)
        for _ in range(args.steps):
            host_step()
            cur.synchronize()                      # the step's result is read on the host
        ev1.record(cur)
        barrier()
        e2e_ms = ev0.elapsed_time(ev1) / args.steps
        h2d = q_h.numel() * q_h.element_size()
        d2h = o_h.numel() * 4 + l_h.numel() * 4
        res["e2e"] = {"value": step_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "api": "dynsplit_decode_step_host_layers (pinned host q/o/lse, one call per step)"}
    if with_dense:
        wsd = D.workspace(D.workspace_bytes(D.OP_DECODE_ATTN, shape, cfg), dev, "decode")

        def dense_step():
            for l in range(L):
                j = l % Ld
                D.decode_attn(wl.qs[j], wl.layers[j], None, out=outs[l], ws=wsd)
        dms, _, _ = time_graph(torch, dense_step, max(2, min(args.steps, 5)), 1, cur, dev, world, barrier)
        dense_bytes = L * B * Hkv * wl.S * 2 * d * e
        res["dense"] = {"ms_per_step": dms, "GB_s": dense_bytes / (dms * 1e-3) / 1e9,
                        "frac_of_peak": dense_bytes / (dms * 1e-3) / 1e9 / peak[0], "sparse_speedup": dms / ms}
    del gstep
    return res


def e2e_model_block(D, G, dev, B=8, S0=32768, outs=(64,), budget=2048):
    """NEXT-4 (the shape of the paper's Fig. 8): ms per generated
    token of a random-weight Llama-3-8B-shaped decoder (32 layers, cuBLAS
    projections) over a 32K synthetic prompt, DynSplit-KV sparse attention
    (the fused layer) vs dense attention (our a9 kernel); one CUDA graph per
    decode step (append, 32 layers, argmax).  The full sweep (B = 1 / 8, 256 /
    1024 / 4096 tokens) is tools/exp_e2e_decode.py."""
    import numpy as np
    import torch
    from paper_2602_03184_b200.model import LlamaShape, RandomLlama, time_decode
    S_cap = S0 + max(outs) + 8
    ids = torch.from_numpy(G.T7_IDS).to(dev)
    res = {}
    for attn in ("sparse", "dense"):
        w10 = torch.from_numpy(np.tile(G.T7_W10, (B, 1))).to(torch.uint8)
        cfg = D.default_config(page_cap=(S_cap // 16) + D.max_blocks(S_cap, D.default_config()) // 2 + 64)
        m = RandomLlama(LlamaShape(), B, S_cap, budget, dev, seed=1, attn=attn, cfg=cfg, delim_ids=ids, w10=w10)
        toks = torch.from_numpy(np.stack([G.tokens(9000 + b, S0) for b in range(B)])).to(dev)
        m.prefill_synthetic(toks, seed=2)
        res[attn] = time_decode(m, toks[:, -1].contiguous(), list(outs))
        assert D.read_device_error(m.ws_app) == 0 and D.read_device_error(m.ws_dec) == 0
        del m
        torch.cuda.empty_cache()
    n = max(outs)
    return {"workload": "NEXT-4: Llama-3-8B-shaped decoder, random bf16 weights, %d sequences, %dK prompt, "
                        "budget %d" % (B, S0 // 1024, budget),
            "generated_tokens": n, "ms_per_token_sparse": res["sparse"][n], "ms_per_token_dense": res["dense"][n],
            "speedup": res["dense"][n] / res["sparse"][n]}


def measured_h2d_gbs(torch, dev, nbytes=1 << 28):
    """Host -> device copy-engine bandwidth from pinned memory (cudaMemcpyAsync,
    256 MiB, best of 10 after 3 warm-up copies): the PCIe / C2C yardstick of
    the offload tier (the zero-copy mover can come close to or above it)."""
    h = torch.ones(nbytes, dtype=torch.uint8).pin_memory()
    dbuf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(3):  # warm-up (first touches, DMA setup)
        dbuf.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dbuf.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del h, dbuf
    return best


def offload_block(args, torch, D, G, dev, cur, barrier, S=32768, L=32, budget=2048, tau=0.9):
    """NEXT-3 (the paper's CPU-GPU deployment, with KV
    Reuse Steps 1-3): config 2's shape (Llama-3-8B decode, 32K,
    budget 2K, one sequence) with every layer's pages in pinned host memory.
    A decode step = per layer a5+a6 on the resident digests, the reuse plan,
    the move of the fresh pages host -> device cache (zero-copy kernel reads
    over PCIe), a7+a8 over the cache (dynsplit_decode_layer_offload), over a
    walk of consecutive queries (q_t = tau q_{t-1} + sqrt(1 - tau^2) z).
    Modes: paper (reuse, truncated to the min over KV heads), reuse without
    truncation, no reuse, and the dense offloaded baseline (every page moved,
    dense attention)."""
    import dataclasses
    Hq, Hkv, d = 32, 8, 128
    wl = Workload(D, G, 1, S, Hq, Hkv, L, 0.0, 4242 + args.seed, dev, args.seed * 7919 + 300)
    cfg, shape = wl.cfg, wl.shape
    offs = []
    for l in range(L):
        offs.append(D.offload_layer(wl.layers[l], budget, Hq))
        wl.layers[l] = None
    torch.cuda.empty_cache()
    T = args.warmup + args.steps
    gen = torch.Generator(device=dev)
    gen.manual_seed(31 + args.seed)
    walks = [G.torch_query_walk(gen, T, wl.qs[l], tau) for l in range(L)]   # [T, 1, Hq, d] per layer
    qb = [torch.empty_like(wl.qs[l]) for l in range(L)]
    outs = [(torch.empty(1, Hq, d, device=dev), torch.empty(1, Hq, device=dev)) for _ in range(L)]
    sel = [D._sel_outputs(shape, cfg, budget, dev, want_blocks=False) for _ in range(L)]
    ws = D.workspace(D.workspace_bytes(D.OP_DECODE_OFFLOAD, shape, cfg, budget), dev, "offload_bench")
    pv = offs[0].layer.page_valid[0].long().cpu()

    def run_mode(truncate, reuse):
        def step():
            for l in range(L):
                _, ns, mg, kp, w = sel[l]
                D.decode_layer_offload(qb[l], offs[l], budget, truncate=truncate, reuse=reuse,
                                       out=(ns, mg, kp, w, outs[l][0], outs[l][1]), ws=ws)
        for l in range(L):
            qb[l].copy_(walks[l][0])
        s2 = torch.cuda.Stream(dev)
        s2.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s2):
            step()
        torch.cuda.current_stream(dev).wait_stream(s2)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        # timed: the walk from an empty cache; steps after the warm-up timed
        for o_ in offs:
            o_.reset()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(T + 1)]
        moved, reused, pages = [], [], []
        for t_ in range(T):
            for l in range(L):
                qb[l].copy_(walks[l][t_])
            evs[t_].record(cur)
            g.replay()
        evs[T].record(cur)
        barrier()
        ms = evs[args.warmup].elapsed_time(evs[T]) / args.steps
        # untimed replay of the same walk: bytes moved per step (valid rows of the fresh pages)
        for o_ in offs:
            o_.reset()
        for t_ in range(T):
            for l in range(L):
                qb[l].copy_(walks[l][t_])
            g.replay()
            if t_ >= args.warmup:
                mb = rb = npg = 0
                for o_ in offs:
                    fc = o_.fetch_count[0].cpu()
                    fl = o_.fetch[0].cpu()
                    for hk in range(Hkv):
                        mb += int(pv[fl[hk, : int(fc[hk]), 0].long()].sum())
                    st = o_.reuse_stats[0].cpu()
                    rb += int(st[:, 0].sum())
                    npg += int(st.sum())
                moved.append(mb * 2 * d * 2)
                reused.append(rb)
                pages.append(npg)
        assert D.read_device_error(ws) == 0
        del g
        return {"ms_per_step": ms, "moved_bytes_per_step": float(np.mean(moved)),
                "pcie_GB_s": float(np.mean(moved)) / (ms * 1e-3) / 1e9,
                "reused_page_frac": float(np.sum(reused)) / max(1, float(np.sum(pages)))}

    res = {"paper_reuse_truncated": run_mode(True, True), "reuse_untruncated": run_mode(False, True),
           "no_reuse": run_mode(True, False)}
    # the fetch kernel alone (the last step's fetch lists, no-reuse mode: every selected page)
    def fetch_only():
        for l in range(L):
            D.fetch_pages(offs[l], Hq)
    fms, _, gf = time_graph(torch, fetch_only, args.steps, args.warmup, cur, dev, 1, barrier)
    del gf
    h2d = measured_h2d_gbs(torch, dev)
    nm = res["no_reuse"]["moved_bytes_per_step"]
    res["fetch_kernel"] = {"bound": "pcie", "achieved": nm / (fms * 1e-3) / 1e9, "unit": "GB/s",
                           "peak": h2d, "frac": nm / (fms * 1e-3) / 1e9 / h2d, "us_per_layer": fms * 1e3 / L,
                           "peak_source": "cudaMemcpyAsync pinned host -> device, 256 MiB, best of 10, measured in this run"}
    # dense offloaded baseline: every page of every layer moved, dense attention (shared device cache)
    mp = D.max_pages(S, cfg)
    Kc = torch.empty(1, Hkv, mp, cfg.page_size, d, dtype=torch.bfloat16, device=dev)
    Vc = torch.empty_like(Kc)
    dls = [dataclasses.replace(offs[l], n_slots=mp, Kc=Kc, Vc=Vc) for l in range(L)]
    wsd = D.workspace(D.workspace_bytes(D.OP_DECODE_ATTN, shape, cfg), dev, "decode")

    def dense_step():
        for l in range(L):
            D.fetch_pages(dls[l], Hq, dense=True)
            D.decode_attn(qb[l], D.cache_view(dls[l]), None, out=outs[l], ws=wsd)
    dms, _, gd = time_graph(torch, dense_step, 2, 1, cur, dev, 1, barrier)
    del gd
    dense_bytes = L * Hkv * S * 2 * d * 2
    res["dense_offload"] = {"ms_per_step": dms, "moved_bytes_per_step": dense_bytes,
                            "pcie_GB_s": dense_bytes / (dms * 1e-3) / 1e9}
    res["speedup_vs_dense_offload"] = dms / res["paper_reuse_truncated"]["ms_per_step"]
    res["workload"] = ("NEXT-3: C2 shape (Llama-3-8B decode, 32 layers, 32Q/8KV) at 32K, budget 2K, 1 sequence, "
                       "KV pages in pinned host memory, query walk tau = %.2f" % tau)
    res["context"] = "paper: 2.4x over full attention in its CPU-GPU deployment (P:473), A800 + PCIe, other models"
    del offs, dls, Kc, Vc
    torch.cuda.empty_cache()
    return res


def cpu_baseline_leg(args, wl: Workload, budget):
    """The oracle on this host's cores: 1 thread, and all cores (forked
    workers over whole KV groups of heads), on a bounded sample (heads of
    layer 0 of sequence 0)."""
    from oracle import dynsplit_oracle as O
    from synth import generators as G
    starts = O.segment(G.tokens(args.seed * 7919 + 0, wl.S), G.T7_IDS, G.T7_W10, 32, 14)
    g = wl.Hq // wl.Hkv
    heads = min(args.cpu_sample_heads, wl.Hq)
    lb = oracle_layer_bytes(wl.q0, wl.K0, starts, budget, wl.Hkv, g)
    out = {}
    cores = cpu_cores()
    groups = heads // g
    with cpu_threads_limit():
        for tag, workers in (("1_thread", 1), ("all_cores", min(cores, groups))):
            ts = []
            t_start = time.perf_counter()
            while not ts or (time.perf_counter() - t_start < args.cpu_seconds / 2 and len(ts) < 20):
                ts.append(time_oracle(wl.q0, wl.K0, wl.V0, starts, budget, heads, workers))
            sec = float(np.mean(ts))
            out[tag] = {"value": lb * heads / wl.Hq / sec / 1e9, "seconds_per_sample": sec, "samples": len(ts),
                        "workers": workers}
    one, allc = out["1_thread"], out["all_cores"]
    return {"value": allc["value"], "unit": "GB/s", "cores": allc["workers"], "kind": "oracle",
            "sample": f"oracle decode step of {heads}/{wl.Hq} heads of layer 0 of sequence 0 at S={wl.S}, "
                      f"budget {budget}; value = {allc['workers']} forked single-thread workers (one per KV "
                      f"group, the parallelism the sample has; the host has {cores} cores), "
                      f"{allc['seconds_per_sample']:.2f} s per sample; 1 thread: {one['value']:.4f} GB/s "
                      f"({one['seconds_per_sample']:.2f} s per sample)",
            "one_thread_value": one["value"], "host_cores": cores, "cpu": cpu_model()}


def run_seqsplit(args, world, rank, local):
    """Config 4 sequence-split across the ranks (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2602_03184_b200 import dynsplit as D
    from paper_2602_03184_b200 import parallel as PAR
    from synth import generators as G
    dev = torch.device("cuda", local)
    S, Hq, Hkv, d, L, budget = args.seq, 40, 40, 128, 40, args.budget
    Ld = min(L, 10)
    cfg = D.default_config()
    toks = torch.from_numpy(G.tokens(args.seed * 7919, S)[None]).to(dev)
    ids = torch.from_numpy(G.T7_IDS).to(dev)
    glob, ranges = PAR.global_plan(toks, ids, cfg, G.T7_W10, Hq, Hkv, world)
    t_lo, t_hi = PAR.shard_token_range(glob.block_starts[0].tolist(), ranges, rank)
    gen = torch.Generator(device=dev)
    layers, qs = [], []
    for l in range(Ld):
        gen.manual_seed(1000003 * (args.seed + 1) + 7 * l + 1)          # q: identical on every rank
        q = torch.randn(1, Hq, d, generator=gen, device=dev).to(torch.bfloat16)
        gen.manual_seed(1000003 * (args.seed + 1) + 7 * l + 2 + 1000 * rank)  # K/V: this rank's tokens
        n_loc = max(t_hi - t_lo, 1)
        K = (1.5 * torch.randn(1, n_loc, Hkv, d, generator=gen, device=dev)).to(torch.bfloat16)
        V = torch.randn(1, n_loc, Hkv, d, generator=gen, device=dev).to(torch.bfloat16)
        layers.append(PAR.local_layer(glob, ranges, rank, K, V, cfg, Hq))
        qs.append(q)
        del K, V
    dec = PAR.SeqSplitDecoder(glob, ranges, rank, Hq, budget, dev)
    o = torch.empty(Hq, d, device=dev)
    lse = torch.empty(Hq, device=dev)

    def step():
        for l in range(L):
            dec.step(qs[l % Ld], layers[l % Ld], o=o, lse=lse)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    step()
    torch.cuda.synchronize()
    # algorithmic bytes of this rank: local digests + local union rows + q + o/lse (+ the exchange)
    nloc = int(layers[0].n_blocks[0])
    _, streamed = D.worklist_rows(dec.sel_out[4], dec.gshape, 1)
    rank_bytes = L * (nloc * Hkv * 2 * d * 2 + int(streamed.sum()) * 2 * d * 2 + Hq * d * 2 + Hq * (d + 1) * 4)
    cur = torch.cuda.current_stream(dev)
    clk = ClockSampler(local)
    clk.__enter__()
    if os.environ.get("DYNSPLIT_BENCH_ONE_GPU") == "1":
        # control-flow check only (gloo stages CUDA collectives through the
        # host, which a CUDA graph cannot capture): eager steps, no timing claim
        for _ in range(args.warmup):
            step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(args.steps):
            step()
        e1.record(cur)
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
    else:
        ms, per, _ = time_graph(torch, step, args.steps, args.warmup, cur, dev, world, barrier)
    clk.__exit__(None, None, None)
    vals = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(rank_bytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms = vals.item()
    if rank == 0:
        peak = measured_peak_hbm()
        line = {"metric": METRIC, "value": tot.item() / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": WORKLOAD_C4, "seq_len": S, "layers": L, "distinct_layer_caches": Ld,
                           "heads_q": Hq, "heads_kv": Hkv, "head_dim": d, "budget": budget,
                           "parallelism": f"sequence-split x{world}", "ranges": ranges,
                           "l2": "no flush: every layer cache >> 126 MB L2"},
                "us_per_layer": ms * 1e3 / L,
                "step_frac_of_peak_aggregate": tot.item() / (ms * 1e-3) / 1e9 / (peak[0] * world),
                "gpu_launches": None, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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

    # DYNSPLIT_BENCH_ONE_GPU=1 (control-flow checks of the multi-rank path on a
    # one-GPU box only; never a timing): every rank on cuda:0, gloo collectives
    one_gpu = os.environ.get("DYNSPLIT_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    D.lib()
    if args.mode == "seqsplit":
        return run_seqsplit(args, world, rank, local)

    B, S, Hq, Hkv, d, L = args.batch_per_gpu, args.seq, args.hq, args.hkv, 128, args.layers
    budget = args.budget
    cur = torch.cuda.current_stream(dev)
    peak = measured_peak_hbm()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if args.only_offload:
        print(json.dumps({"offload": offload_block(args, torch, D, G, dev, cur, barrier)}), flush=True)
        return

    # ---- the headline block: config 3's per-GPU shard, every layer its own cache
    wl = Workload(D, G, B, S, Hq, Hkv, L, args.rho, 1000003 * (args.seed + 1) + rank, dev,
                  args.seed * 7919 + rank * B)
    clk = ClockSampler(local)
    clk.__enter__()
    main_res = decode_block(args, torch, D, wl, L, budget, dev, cur, world, barrier, peak,
                            with_three_kernel=(world == 1))
    clk.__exit__(None, None, None)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(args, wl, budget)
    # NEXT-2 variants on the same workload (paper variants, DESIGN R23 / R24):
    # group-shared GQA selection and the whole-block budget (context keys)
    variants = {}
    if world == 1 and not args.no_extra:
        import copy
        for name, fields in (("gqa_group_shared", {"gqa_mode": 1}), ("whole_block_budget", {"budget_mode": 1})):
            saved = [lay.cfg for lay in wl.layers]
            cfg_v = copy.copy(wl.cfg)
            for k2, v2 in fields.items():
                setattr(cfg_v, k2, v2)
            for lay in wl.layers:
                lay.cfg = cfg_v
            wl_cfg = wl.cfg
            wl.cfg = cfg_v
            try:
                rv = decode_block(args, torch, D, wl, L, budget, dev, cur, world, barrier, peak, with_e2e=False,
                                  with_dense=False)
            finally:
                wl.cfg = wl_cfg
                for lay, c0 in zip(wl.layers, saved):
                    lay.cfg = c0
            variants[name] = {"ms_per_step": rv["ms_per_step"], "GB_s": rv["GB_s"],
                              "frac_of_peak": rv["roofline"]["frac"], "union_factor": rv["union_factor"],
                              "bytes_per_step": rv["bytes_per_step"], "config": fields}
    del wl
    torch.cuda.empty_cache()

    # ---- max over ranks of the headline
    vals = torch.tensor([main_res["ms_per_step"], main_res["e2e"]["ms_per_step"]], dtype=torch.float64, device=dev)
    tot = torch.tensor([main_res["bytes_per_step"]], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    step_ms, e2e_ms = vals.tolist()
    all_bytes = tot.item()

    # ---- more configurations of the metric on one GPU (N = 1 only)
    extra = {}
    if world == 1 and not args.no_extra:
        wl8 = Workload(D, G, 8, S, Hq, Hkv, 8, args.rho, 77 + args.seed, dev, args.seed * 7919 + 100)
        r8 = decode_block(args, torch, D, wl8, L, budget, dev, cur, world, barrier, peak)
        r8["config"] = {"workload": "C3 unsharded: Llama-3-8B decode, 8 sequences on 1 GPU, 128K, budget 4K",
                        "batch": 8, "layers": L, "distinct_layer_caches": 8,
                        "note": "32 layers of work over 8 distinct layer caches (each 5.2 GB >> L2)"}
        extra["c3_b8"] = r8
        del wl8
        torch.cuda.empty_cache()
        wl4 = Workload(D, G, 1, S, 40, 40, 10, args.rho, 99 + args.seed, dev, args.seed * 7919 + 200)
        r4 = decode_block(args, torch, D, wl4, 40, budget, dev, cur, world, barrier, peak)
        r4["config"] = {"workload": "C4 on 1 GPU: Llama2-13B decode (40 layers, 40 MHA heads), 128K, budget 4K",
                        "layers": 40, "distinct_layer_caches": 10,
                        "note": "40 layers of work over 10 distinct layer caches (each 3.4 GB >> L2)"}
        extra["c4"] = r4
        del wl4
        torch.cuda.empty_cache()

        if not args.no_e2e_model:
            extra["e2e_model"] = e2e_model_block(D, G, dev)
            torch.cuda.empty_cache()
        if not args.no_offload:
            extra["offload"] = offload_block(args, torch, D, G, dev, cur, barrier)

    prefill = None
    if rank == 0 and not args.no_prefill:
        prefill = prefill_c5(args, D, G, D.default_config(), torch.from_numpy(G.T7_IDS).to(dev), dev, cur)

    if rank == 0:
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
                       "budget": budget, "rho": args.rho, "C": 32, "delta": 14, "page_size": 16,
                       "parallelism": f"batch-shard x{world}",
                       "l2": "no flush: ~%.0f MiB touched per step >> 126 MB L2" %
                             (main_res["bytes_per_step"] / 2 ** 20)},
            "us_per_step": step_ms * 1e3,
            "us_per_layer": step_ms * 1e3 / L,
            "step_ms_p10_p50_p90": main_res["step_ms_p10_p50_p90"],
            "bytes_per_step": main_res["bytes_per_step"],
            "union_factor": main_res["union_factor"],
            "roofline": main_res["roofline"],
            "e2e": dict(main_res["e2e"], value=all_bytes / (e2e_ms * 1e-3) / 1e9, ms_per_step=e2e_ms),
            "gpu_launches": main_res["fused_launches_per_step"] * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        if "dense" in main_res:
            line["dense"] = main_res["dense"]
        if "three_kernel_path" in main_res:
            line["three_kernel_path"] = main_res["three_kernel_path"]
        line.update(extra)
        if variants:
            line["variants"] = variants
        if prefill:
            line["prefill"] = prefill
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Phase timeline of the fused decode layer (k_decode_fused) inside a CUDA
graph of L layers, from the debug build's %globaltimer stamps (last layer's
launch is the last writer of the stamp buffer).

    DYNSPLIT_DEBUG_BUILD=1 python tools/exp_fused_timeline.py [budget] [B] [Hq] [Hkv]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

assert os.environ.get("DYNSPLIT_DEBUG_BUILD"), "needs the debug build"
dev = torch.device("cuda:0")
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
Hq = int(sys.argv[3]) if len(sys.argv) > 3 else 32
Hkv = int(sys.argv[4]) if len(sys.argv) > 4 else 8
S, d, L = 131072, 128, 4
cfg = D.default_config()
gen = torch.Generator(device=dev)
gen.manual_seed(1)
toks = torch.from_numpy(np.stack([G.tokens(b, S) for b in range(B)])).to(dev)
ids = torch.from_numpy(G.T7_IDS).to(dev)
layers, qs = [], []
for _ in range(L):
    q, K, V = G.torch_decode_layer(gen, S, Hq, Hkv, d, B, dev)
    layers.append(D.build_blocks(toks, ids, K, V, cfg, static_w10=G.T7_W10, Hq=Hq))
    qs.append(q.contiguous())
    del K, V
shape = D.make_shape(B, S, Hq, Hkv, d)
sels = [D._sel_outputs(shape, cfg, budget, dev, want_blocks=False) for _ in range(L)]
outs = [(torch.empty(B, Hq, d, device=dev), torch.empty(B, Hq, device=dev)) for _ in range(L)]
ws = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "layer")
lib = D.lib()
NAMES = ["start", "plan", "pdl_wait", "scored+arrive A", "A passed", "range classified", "B passed+gathered",
         "band selected", "bits final", "union counted", "dealt", "pages done", "merged", "B passed", "q loaded", "digests in smem"]


def step():
    for l in range(L):
        _, ns, mg, kp, wl = sels[l]
        D.decode_layer(qs[l], layers[l], budget, out=(ns, mg, kp, wl, outs[l][0], outs[l][1]), ws=ws)


step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    step()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
ncta = 148
print(f"Hq {Hq} Hkv {Hkv}")
dbg = torch.zeros(ncta * 64, dtype=torch.int64, device=dev)
lib.dynsplit_debug_fused_timer.argtypes = [ctypes.c_void_p]
lib.dynsplit_debug_fused_timer(ctypes.c_void_p(dbg.data_ptr()))
g.replay()
torch.cuda.synchronize()
lib.dynsplit_debug_fused_timer(ctypes.c_void_p(0))
tc = dbg.view(ncta, 64).cpu().numpy().astype(np.float64)
used = tc[:, 0] > 0
t = tc[used, :16]
clk = tc[used, 16:]
t0 = t[:, 0].min()
print(f"CTAs stamped: {used.sum()}  budget {budget}  B {B}")
ORDER = [0, 1, 2, 14, 15, 3, 4, 5, 13, 7, 8, 9, 10, 11, 12]
prev = None
for k in ORDER:
    name = NAMES[k]
    col = t[:, k]
    col = col[col > 0]
    if len(col) == 0:
        continue
    r = (col - t0) / 1e3
    mhz = ""
    if prev is not None:
        ok = (t[:, k] > 0) & (t[:, prev] > 0)
        dt = t[ok, k] - t[ok, prev]
        dc = clk[ok, k] - clk[ok, prev]
        if dt.sum() > 0:
            mhz = f"  SM clock over the phase {dc.sum() / dt.sum() * 1e3:6.0f} MHz, {np.median(dc):8.0f} cycles p50"
    print(f"{k:2d} {name:18s} n={len(col):3d}  min {r.min():7.2f}  p50 {np.median(r):7.2f}  max {r.max():7.2f} us{mhz}")
    prev = k
# extra %globaltimer stamps (thread 0): 56 + k
XN = {4: "bounds ready", 5: "classified (loop)", 6: "gathered (warp 0)", 7: "band-selected (warp 0)"}
tx = tc[used, 56:64]
for k, name in XN.items():
    col = tx[:, k]
    col = col[col > 0]
    if len(col):
        r = (col - t0) / 1e3
        print(f"x{k} {name:22s} n={len(col):3d}  min {r.min():7.2f}  p50 {np.median(r):7.2f}  max {r.max():7.2f} us")
# fast-path diagnostics of each group's split 0 (debug slots 32 + 4 g ..: band entries, overflow, W_hi, W_bd)
if os.environ.get("DYNSPLIT_TL_DIAG"):
    dg = tc[:, 32:48].astype(np.int64)
    for c in range(0, int(used.sum()), max(1, int(used.sum()) // (B * Hkv))):
        print("group CTA", c, [tuple(dg[c, 4 * g:4 * g + 4]) for g in range(4)], "budget", budget)
# per-layer time from the graph
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    g.replay()
ev[1].record()
torch.cuda.synchronize()
print(f"step of {L} layers: {ev[0].elapsed_time(ev[1]) / 20 * 1e3:.1f} us ({ev[0].elapsed_time(ev[1]) / 20 / L * 1e3:.2f} us/layer)")

"""Timeline of one decode layer (a5 score -> a6 select -> a7/a8 attention) as
it runs inside the CUDA graph of a 4-layer step, from the debug build's
%globaltimer stamps (resolution ~0.25 us).  Layer 3's kernels are the last
writers of each stamp buffer.

    DYNSPLIT_DEBUG_BUILD=1 python tools/exp_step_timeline.py [budget]
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
B, S, Hq, Hkv, d, L = 1, 131072, 32, 8, 128, 4
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = D.default_config()
gen = torch.Generator(device=dev)
gen.manual_seed(1)
toks = torch.from_numpy(G.tokens(0, S)[None]).to(dev)
ids = torch.from_numpy(G.T7_IDS).to(dev)
layers, qs = [], []
for _ in range(L):
    q, K, V = G.torch_decode_layer(gen, S, Hq, Hkv, d, B, dev)
    layers.append(D.build_blocks(toks, ids, K, V, cfg, static_w10=G.T7_W10, Hq=Hq))
    qs.append(q.contiguous())
    del K, V
shape = D.make_shape(B, S, Hq, Hkv, d)
mb = D.max_blocks(S, cfg)
scores = [torch.empty(B, Hq, mb, device=dev) for _ in range(L)]
sels = [D._sel_outputs(shape, cfg, budget, dev, want_blocks=False) for _ in range(L)]
outs = [(torch.empty(B, Hq, d, device=dev), torch.empty(B, Hq, device=dev)) for _ in range(L)]
ws_sel = D.workspace(D.workspace_bytes(D.OP_SELECT, shape, cfg, budget), dev, "select")
ws_dec = D.workspace(D.workspace_bytes(D.OP_DECODE_ATTN, shape, cfg), dev, "decode")


FUSED = True  # dynsplit_select (a5 + a6 through one ABI call)
# TL_MODE=layer: dynsplit_decode_layer per layer; default: dynsplit_select +
# dynsplit_decode_attn
LAYER = os.environ.get("TL_MODE") == "layer"
ws_lay = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "layer")


def step():
    for l in range(L):
        if LAYER:
            _, ns, mg, kp, wl = sels[l]
            D.decode_layer(qs[l], layers[l], budget, out=(ns, mg, kp, wl, outs[l][0], outs[l][1]), ws=ws_lay)
            continue
        if FUSED:
            sb, ns, mg, kp, wl = sels[l]
            D.select(qs[l], layers[l], budget, out=(sb, ns, mg, kp, wl, None), ws=ws_sel)
        else:
            D.score_blocks(qs[l], layers[l], out=scores[l])
            D.select_from_scores(scores[l], layers[l], budget, Hq, out=sels[l], ws=ws_sel)
        D.decode_attn(qs[l], layers[l], sels[l][4], out=outs[l], ws=ws_dec)


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
lib = D.lib()
bufs = {k: torch.zeros(n, dtype=torch.int64, device=dev) for k, n in
        [("score", 4096 * 4), ("select", 4096 * 16), ("attn", 4096 * 8)]}
for k in bufs:
    getattr(lib, f"dynsplit_debug_{k}_timer").argtypes = [ctypes.c_void_p]
    getattr(lib, f"dynsplit_debug_{k}_timer")(ctypes.c_void_p(bufs[k].data_ptr()))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
g.replay()
b.record()
torch.cuda.synchronize()
for k in bufs:
    getattr(lib, f"dynsplit_debug_{k}_timer")(ctypes.c_void_p(0))
print(f"step (4 layers, debug build) {a.elapsed_time(b) * 1e3:.1f} us")
sc = bufs["score"].view(-1, 4).cpu().numpy().astype(np.float64)
sc = sc[sc[:, 0] > 0]
t0 = sc[:, 0].min()


def show(name, arr, cols):
    for k, n in enumerate(cols):
        if n is None:
            continue
        v = arr[:, k]
        v = v[v > 0]
        if len(v) == 0:
            continue
        r = (v - t0) / 1e3
        print(f"{name:7s} {n:13s} n={len(r):4d} min {r.min():7.2f} p50 {np.median(r):7.2f} max {r.max():7.2f} us")


show("score", sc, ["start", "pdl_wait", "end", "digests_in"])
se = bufs["select"].view(-1, 16).cpu().numpy().astype(np.float64)
se = se[se[:, 0] > 0]
show("select", se, ["start", "plan", "pdl_wait", "keys", "threshold", "bits+arrive", "wait+peers",
                    "union_scan", "writes", "final_wait", "first_key"])
at = bufs["attn"].view(-1, 8).cpu().numpy().astype(np.float64)
at = at[at[:, 0] > 0]
show("attn", at, ["start", "pdl_wait", "first_page", "consumed", "partial", "merged", "entries+cnt", "issued"])

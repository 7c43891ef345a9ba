"""Per-layer time of the fused decode layer in a CUDA graph of L layers
(release build; DYNSPLIT_LIB_AB=<file in lib/> times another build):
    python tools/time_fused.py [S] [B] [budget] [L] [Hq] [Hkv]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

S, B, budget, L, Hq, Hkv = [int(x) for x in (sys.argv[1:] + ["131072", "1", "4096", "8", "32", "8"][len(sys.argv) - 1:])]
dev = torch.device("cuda:0")
d = 128
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


def step():
    for l in range(L):
        _, ns, mg, kp, wl = sels[l]
        D.decode_layer(qs[l], layers[l], budget, out=(ns, mg, kp, wl, outs[l][0], outs[l][1]), ws=ws)


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
res = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 50 / L * 1e3)
print(f"{os.environ.get('DYNSPLIT_LIB_AB', 'libdynsplit.so')}: S {S} B {B} budget {budget}: "
      f"Hq {Hq} Hkv {Hkv}: {np.median(res):.2f} us/layer (min {min(res):.2f}), err {D.read_device_error(ws)}", flush=True)

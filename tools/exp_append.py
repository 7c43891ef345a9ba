"""NEXT-1 timing (not part of the product): decode-time append at the C3
shape.  A 128K prefix is planned and paged through the append path, then
one token per step is appended to 32 layers (plan once + K/V per layer),
captured in a CUDA graph.  python tools/exp_append.py [L0] [layers]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

dev = torch.device("cuda:0")
L0 = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
NL = int(sys.argv[2]) if len(sys.argv) > 2 else 32
B, Hq, Hkv, d = 1, 32, 8, 128
steps = 64
S_cap = L0 + steps + 8
cfg = D.default_config()
toks = torch.from_numpy(G.tokens(0, S_cap)[None]).to(dev)
ids = torch.from_numpy(G.T7_IDS).to(dev)
w10 = torch.from_numpy(np.tile(G.T7_W10, (B, 1))).to(dev)
gen = torch.Generator(device=dev)
gen.manual_seed(5)
K = (1.5 * torch.randn(B, S_cap, Hkv, d, generator=gen, device=dev)).to(torch.bfloat16)
V = torch.randn(B, S_cap, Hkv, d, generator=gen, device=dev).to(torch.bfloat16)
layers = [D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, torch.bfloat16, dev)]
for _ in range(NL - 1):
    layers.append(D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, torch.bfloat16, dev, plan_from=layers[0]))
ws = D.append_workspace(layers[0])

a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
D.append_plan(toks, ids, layers[0], 0, L0, ws)
b.record()
torch.cuda.synchronize()
t_plan0 = a.elapsed_time(b)
a.record()
D.append_kv(layers[0], K[:, :L0].contiguous(), V[:, :L0].contiguous(), 0, L0, ws)
b.record()
torch.cuda.synchronize()
t_kv0 = a.elapsed_time(b)
for l in range(1, NL):
    D.append_kv(layers[l], K[:, :L0].contiguous(), V[:, :L0].contiguous(), 0, L0, ws)
torch.cuda.synchronize()
print(f"prefix {L0} through the append path: plan {t_plan0:.2f} ms, K/V of one layer {t_kv0:.2f} ms")

Kn = [K[:, L0 + i: L0 + i + 1].contiguous() for i in range(steps)]
Vn = [V[:, L0 + i: L0 + i + 1].contiguous() for i in range(steps)]


def step(i):
    Lp = L0 + i
    D.append_plan(toks, ids, layers[0], Lp, Lp + 1, ws)
    D.append_kv_layers(layers, [Kn[i]] * NL, [Vn[i]] * NL, Lp, Lp + 1, ws)


# graph of `steps` consecutive one-token steps (each step depends on the previous plan)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(steps):
        step(i)
a.record()
g.replay()
b.record()
torch.cuda.synchronize()
print(f"one-token append, plan + K/V of {NL} layers: {a.elapsed_time(b) * 1e3 / steps:.1f} us per step "
      f"(n_blocks {int(layers[0].n_blocks[0])})")

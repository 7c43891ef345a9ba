"""One fused decode layer at a chosen shape for ncu source-level profiling:
    python tools/ncu_fused_case.py S B budget force
(force: 0 = normal paths, 1 = every head through the histogram fallback,
2 = every head through the CTA-wide slow path).  Runs 3 launches; profile the
third with  ncu -k regex:k_decode_fused --launch-skip 2 --launch-count 1."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

S, B, budget, force = (int(x) for x in sys.argv[1:5])
dev = torch.device("cuda:0")
Hq, Hkv, d = 32, 8, 128
cfg = D.default_config()
gen = torch.Generator(device=dev)
gen.manual_seed(1)
toks = torch.from_numpy(np.stack([G.tokens(b, S) for b in range(B)])).to(dev)
q, K, V = G.torch_decode_layer(gen, S, Hq, Hkv, d, B, dev)
layer = D.build_blocks(toks, torch.from_numpy(G.T7_IDS).to(dev), K, V, cfg, static_w10=G.T7_W10, Hq=Hq)
del K, V
lib = D.lib()
lib.dynsplit_debug_fused_force(force)
shape = D.make_shape(B, S, Hq, Hkv, d)
_, ns, mg, kp, wl = D._sel_outputs(shape, cfg, budget, dev, want_blocks=False)
o, lse = torch.empty(B, Hq, d, device=dev), torch.empty(B, Hq, device=dev)
ws = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "ncu")
for _ in range(3):
    D.decode_layer(q.contiguous(), layer, budget, out=(ns, mg, kp, wl, o, lse), ws=ws)
torch.cuda.synchronize()
lib.dynsplit_debug_fused_force(0)
print("ok", D.read_device_error(ws))

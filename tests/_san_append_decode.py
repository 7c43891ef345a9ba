"""Subprocess body of test_gpu_errors.test_fused_synccheck: the decode-model
flow (append_plan_dev -> append_kv_layers_dev -> decode_layer, the kv-append
kernel's shared memory left behind for the fused kernel) on a capacity layer,
small enough for compute-sanitizer.  Prints "ok" when the outputs are finite
and the device error words are clear."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

dev = torch.device("cuda:0")
B, S0, S_cap, Hq, Hkv = 1, 3000, 3100, 32, 8
cfg = D.default_config()
ids = torch.from_numpy(G.T7_IDS).to(dev)
w10 = torch.from_numpy(np.tile(G.T7_W10, (B, 1))).to(torch.uint8).to(dev)
lay = D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, torch.bfloat16, dev)
ws = D.append_workspace(lay)
tokens = torch.zeros(B, S_cap, dtype=torch.int32, device=dev)
tokens[:, :S0] = torch.from_numpy(np.stack([G.tokens(77 + b, S0) for b in range(B)])).to(dev)
g = torch.Generator(device=dev)
g.manual_seed(3)
K = (1.5 * torch.randn(B, S0, Hkv, 128, generator=g, device=dev)).to(torch.bfloat16)
V = torch.randn(B, S0, Hkv, 128, generator=g, device=dev).to(torch.bfloat16)
D.append_plan(tokens, ids, lay, 0, S0, ws)
D.append_kv(lay, K, V, 0, S0, ws)
pos = torch.full((1,), S0, dtype=torch.int32, device=dev)
shape = D.make_shape(B, S_cap, Hq, Hkv, 128)
budget = 512
wsd = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "san")
_, ns, mg, kp, wl = D._sel_outputs(shape, cfg, budget, dev, want_blocks=False)
o = torch.empty(B, Hq, 128, device=dev)
lse = torch.empty(B, Hq, device=dev)
for i in range(3):
    tokens[:, S0 + i] = 5 + i
    D.append_plan_dev(tokens, ids, lay, pos, 1, ws)
    kn = torch.randn(B, 1, Hkv, 128, generator=g, device=dev).to(torch.bfloat16)
    D.append_kv_layers_dev([lay], [kn], [kn.clone()], pos, 1, ws)
    q = torch.randn(B, Hq, 128, generator=g, device=dev).to(torch.bfloat16)
    D.decode_layer(q, lay, budget, out=(ns, mg, kp, wl, o, lse), ws=wsd)
    pos.add_(1)
torch.cuda.synchronize()
assert D.read_device_error(ws) == 0 and D.read_device_error(wsd) == 0
assert torch.isfinite(o).all() and torch.isfinite(lse).all()
print("ok", flush=True)

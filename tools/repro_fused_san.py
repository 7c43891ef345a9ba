"""Sanitizer repro: append (plan / kv) then the fused decode on a capacity layer."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D
from paper_2602_03184_b200.model import LlamaShape, RandomLlama
from synth import generators as G
mode = sys.argv[1]
S0, S_cap, B = 4096, 8200, 1
dev = torch.device("cuda:0")
ids = torch.from_numpy(G.T7_IDS).to(dev)
w10 = torch.from_numpy(np.tile(G.T7_W10, (B, 1))).to(torch.uint8)
cfg = D.default_config(page_cap=(S_cap // 16) + D.max_blocks(S_cap, D.default_config()) // 2 + 64)
m = RandomLlama(LlamaShape(layers=1, vocab=32000, d_model=256, ffn=512), B, S_cap, 2048, dev, seed=1, cfg=cfg,
                delim_ids=ids, w10=w10)
toks = torch.from_numpy(np.stack([G.tokens(9000 + b, S0) for b in range(B)])).to(dev)
m.prefill_synthetic(toks, seed=2)
torch.cuda.synchronize()
lay = m.layers[0]
q = torch.randn(B, 32, 128, device=dev).to(torch.bfloat16)
k = torch.randn(B, 1, 8, 128, device=dev).to(torch.bfloat16)
if "p" in mode:
    m.tokens[:, S0] = 5
    D.append_plan_dev(m.tokens, m.delim_ids, lay, m.pos, 1, m.ws_app)
    torch.cuda.synchronize(); print("plan ok", lay.n_blocks.tolist(), flush=True)
saved = (lay.digests.clone(), lay.Kp.clone(), lay.Vp.clone())
if "k" in mode:
    D.append_kv_layers_dev([lay], [k], [k.clone()], m.pos, 1, m.ws_app)
    torch.cuda.synchronize(); print("kv ok", flush=True)
if "D" in mode:
    lay.digests.copy_(saved[0])
if "K" in mode:
    lay.Kp.copy_(saved[1]); lay.Vp.copy_(saved[2])
if "Z" in mode:
    lay.digests.zero_()
if "x" in mode:
    m.pos.add_(1)
D.decode_layer(q, lay, 2048, out=(m.ns, m.mg, m.kp, m.wl, m.o, m.lse), ws=m.ws_dec)
torch.cuda.synchronize()
print("decode ok", D.read_device_error(m.ws_dec), flush=True)

"""Per-CTA timeline of the decode attention kernel (debug %globaltimer stamps)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

dev = torch.device("cuda:0")
B, S, Hq, Hkv, d = 1, 131072, 32, 8, 128
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = D.default_config()
gen = torch.Generator(device=dev)
gen.manual_seed(1)
toks = torch.from_numpy(G.tokens(0, S)[None]).to(dev)
ids = torch.from_numpy(G.T7_IDS).to(dev)
layers, qs = [], []
for l in range(4):
    q, K, V = G.torch_decode_layer(gen, S, Hq, Hkv, d, B, dev)
    layers.append(D.build_blocks(toks, ids, K, V, cfg, static_w10=G.T7_W10, Hq=Hq))
    qs.append(q)
    del K, V
sels = [D.select(qs[l], layers[l], budget) for l in range(4)]
dbg = torch.zeros(4096 * 8, dtype=torch.int64, device=dev)
lib = D.lib()
lib.dynsplit_debug_attn_timer.argtypes = [ctypes.c_void_p]
for l in range(4):
    D.decode_attn(qs[l], layers[l], sels[l].worklist)
torch.cuda.synchronize()
if os.environ.get("NOCOMPUTE"):
    lib.dynsplit_debug_attn_nocompute(1)
if os.environ.get("NOLOAD"):
    lib.dynsplit_debug_attn_noload(1)
pages = torch.zeros(512, dtype=torch.int64, device=dev)
lib.dynsplit_debug_attn_pages.argtypes = [ctypes.c_void_p]
lib.dynsplit_debug_attn_pages(ctypes.c_void_p(pages.data_ptr()))
lib.dynsplit_debug_attn_timer(ctypes.c_void_p(dbg.data_ptr()))
D.decode_attn(qs[3], layers[3], sels[3].worklist)   # layer 3: its KV is not in L2 (0..2 ran after it)
torch.cuda.synchronize()
lib.dynsplit_debug_attn_timer(ctypes.c_void_p(0))
lib.dynsplit_debug_attn_nocompute(0)
lib.dynsplit_debug_attn_noload(0)
t = dbg.view(-1, 8).cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["start", "pdl_wait", "first_page", "consumed", "partial", "merged"]
for k, n in enumerate(names):
    v = t[:, k]
    v = v[v > 0]
    r = (v - t0) / 1e3
    print(f"{n:11s} n={len(r):4d} min {r.min():7.2f} p50 {np.median(r):7.2f} p90 {np.percentile(r, 90):7.2f} max {r.max():7.2f} us")
pg = pages.cpu().numpy().astype(np.float64)
t_ref = dbg.view(-1, 8).cpu().numpy()[0, 0]
for i in range(64):
    if pg[2 * i] > 0:
        print(f"page {i:2d} warp {i % 4}: wait-start {(pg[2*i]-t_ref)/1e3:6.2f} arrived {(pg[2*i+1]-t_ref)/1e3:6.2f} done {(pg[2*(64+i)]-t_ref)/1e3:6.2f}")
lib.dynsplit_debug_attn_pages(ctypes.c_void_p(0))
_, rows = D.worklist_rows(sels[3].worklist, D.make_shape(B, S, Hq, Hkv), Hq // Hkv)
print("union rows per kv head:", rows.tolist())

"""Phase timeline of the select kernel via in-kernel %globaltimer stamps
(debug instrumentation): python tools/exp_select_phases.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

dev = torch.device("cuda:0")
B, S, Hq, Hkv, d, budget = 1, 131072, 32, 8, 128, 4096
cfg = D.default_config()
gen = torch.Generator(device=dev)
gen.manual_seed(1)
toks = torch.from_numpy(G.tokens(0, S)[None]).to(dev)
ids = torch.from_numpy(G.T7_IDS).to(dev)
q, K, V = G.torch_decode_layer(gen, S, Hq, Hkv, d, B, dev)
layer = D.build_blocks(toks, ids, K, V, cfg, static_w10=G.T7_W10, Hq=Hq)
del K, V
sc = D.score_blocks(q, layer)
dbg = torch.zeros(B * Hkv * 4 * 16, dtype=torch.int64, device=dev)
lib = D.lib()
lib.dynsplit_debug_select_timer.argtypes = [ctypes.c_void_p]
for rep in range(3):
    D.select_from_scores(sc, layer, budget, Hq)
torch.cuda.synchronize()
lib.dynsplit_debug_select_timer(ctypes.c_void_p(dbg.data_ptr()))
D.select_from_scores(sc, layer, budget, Hq)
torch.cuda.synchronize()
lib.dynsplit_debug_select_timer(ctypes.c_void_p(0))
t = dbg.view(-1, 16).cpu().numpy()[:, :10].astype(np.float64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = ["start", "lens", "pdl_wait", "keys+total", "threshold", "csync1", "union_sumk", "scan", "csync2+writes", "csync3"] if os.environ.get("DYNSPLIT_SELECT_GENERIC") else ["start", "plan", "pdl_wait", "keys", "threshold", "bits+arrive", "wait+peers", "union_scan", "writes", "final_wait"]
for k, n in enumerate(names):
    print(f"{n:14s} min {rel[:, k].min():7.2f} med {np.median(rel[:, k]):7.2f} max {rel[:, k].max():7.2f} us")

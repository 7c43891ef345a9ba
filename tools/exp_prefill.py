"""Prefill timing (not part of the product): a1 delimiter scoring and the
whole build (a1-a4) at C5-like shapes.  python tools/exp_prefill.py [S]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

dev = torch.device("cuda:0")
S = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
B, Hq, Hkv, d = 1, 32, 8, 128
cfg = D.default_config()
toks = torch.from_numpy(G.tokens(0, S)[None]).to(dev)
ids = torch.from_numpy(G.T7_IDS).to(dev)
gen = torch.Generator(device=dev)
gen.manual_seed(3)
Qs = (torch.randn(1, B, S, Hq, d, generator=gen, device=dev)).to(torch.bfloat16)
Ks = (torch.randn(1, B, S, Hkv, d, generator=gen, device=dev)).to(torch.bfloat16)
s = D.score_delimiters(toks, ids, Qs, Ks, cfg)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
a.record()
for _ in range(reps):
    D.score_delimiters(toks, ids, Qs, Ks, cfg)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
cand = torch.isin(toks[0, :-1], ids).cpu().numpy()
tk = toks[0].cpu().numpy()
need = np.zeros(S, bool)
for i in np.nonzero(cand)[0]:
    need[i + 1: min(i + 9, S)] = True
rows = np.nonzero(need)[0]
flop = 2 * d * Hq * float(np.sum(rows + 1))
exps = Hq * float(np.sum(rows + 1))
print(f"S={S}: a1 score_delimiters {ms:.2f} ms; needed rows {len(rows)} ({len(rows)/S:.2f}); "
      f"{flop/ms/1e9:.1f} TFLOP/s on the causal QK^T of needed rows, {exps/ms/1e6:.2f} Gexp/s... x1e3 -> "
      f"{exps/(ms*1e-3)/1e12:.2f} Texp/s")

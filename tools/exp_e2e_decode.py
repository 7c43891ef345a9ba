"""NEXT-4 measurement (the shape of the paper's Fig. 8): decode
latency per generated token of a random-weight Llama-3-8B-shaped model at a
32K-token synthetic prompt, DynSplit-KV sparse attention (budget 2048, the
fused layer) vs dense attention (our a9 kernel), over 256 / 1024 / 4096
generated tokens, batch 1 and 8.  One JSON line per configuration.

    python tools/exp_e2e_decode.py [--batches 1,8] [--outs 256,1024,4096] [--prompt 32768]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from paper_2602_03184_b200.model import LlamaShape, RandomLlama, time_decode  # noqa: E402
from synth import generators as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,8")
ap.add_argument("--outs", default="256,1024,4096")
ap.add_argument("--prompt", type=int, default=32768)
ap.add_argument("--budget", type=int, default=2048)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--attn", default="sparse,dense")
args = ap.parse_args()
dev = torch.device("cuda:0")
outs = [int(x) for x in args.outs.split(",")]
S0 = args.prompt
S_cap = S0 + max(outs) + 8
ids = torch.from_numpy(G.T7_IDS).to(dev)
for B in [int(x) for x in args.batches.split(",")]:
    res = {}
    for attn in args.attn.split(","):
        w10 = torch.from_numpy(np.tile(G.T7_W10, (B, 1))).to(torch.uint8)
        cfg = D.default_config(page_cap=(S_cap // 16) + D.max_blocks(S_cap, D.default_config()) // 2 + 64)
        m = RandomLlama(LlamaShape(layers=args.layers), B, S_cap, args.budget, dev, seed=1, attn=attn, cfg=cfg,
                        delim_ids=ids, w10=w10)
        toks = torch.from_numpy(np.stack([G.tokens(9000 + b, S0) for b in range(B)])).to(dev)
        m.prefill_synthetic(toks, seed=2)
        first = toks[:, -1].contiguous()
        res[attn] = time_decode(m, first, outs)
        assert D.read_device_error(m.ws_app) == 0 and D.read_device_error(m.ws_dec) == 0
        del m
        torch.cuda.empty_cache()
    line = {"experiment": "NEXT-4 e2e decode (Fig. 8 shape)", "model": "Llama-3-8B shape, random bf16 weights",
            "batch": B, "prompt_tokens": S0, "budget": args.budget,
            "ms_per_token": {str(n): dict({a: res[a][n] for a in res},
                                          **({"speedup": res["dense"][n] / res["sparse"][n]} if len(res) == 2 else {}))
                             for n in outs},
            "note": "mean ms per generated token up to n tokens (the cache grows from the prompt); one CUDA "
                    "graph per decode step (append, 32 layers, argmax)"}
    print(json.dumps(line), flush=True)

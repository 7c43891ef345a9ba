"""Decode-path timing experiments (not part of the product): per-kernel-group
CUDA-graph timings over L distinct layer caches at 128K, for several budgets.

    python tools/exp_decode.py [--layers 4] [--budgets 16,1024,4096]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402


def time_graph(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--budgets", default="16,1024,4096,16384")
    ap.add_argument("--batch", type=int, default=1)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    B, S, Hq, Hkv, d, L = args.batch, args.seq, 32, 8, 128, args.layers
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
    mb = D.max_blocks(S, cfg)
    scores = [torch.empty(B, Hq, mb, device=dev) for _ in range(L)]
    for budget in [int(x) for x in args.budgets.split(",")]:
        sels = [D._sel_outputs(shape, cfg, budget, dev, want_blocks=False) for _ in range(L)]
        outs = [(torch.empty(B, Hq, d, device=dev), torch.empty(B, Hq, device=dev)) for _ in range(L)]
        ws_sel = D.workspace(D.workspace_bytes(D.OP_SELECT, shape, cfg, budget), dev, "select")
        ws_dec = D.workspace(D.workspace_bytes(D.OP_DECODE_ATTN, shape, cfg), dev, "decode")

        def score():
            for l in range(L):
                D.score_blocks(qs[l], layers[l], out=scores[l])

        def selfs():
            for l in range(L):
                D.select_from_scores(scores[l], layers[l], budget, Hq, out=sels[l], ws=ws_sel)

        def attn():
            for l in range(L):
                D.decode_attn(qs[l], layers[l], sels[l][4], out=outs[l], ws=ws_dec)

        def full():  # the step as two kernels a5 | a6 per layer, interleaved with a7
            for l in range(L):
                D.score_blocks(qs[l], layers[l], out=scores[l])
                D.select_from_scores(scores[l], layers[l], budget, Hq, out=sels[l], ws=ws_sel)
                D.decode_attn(qs[l], layers[l], sels[l][4], out=outs[l], ws=ws_dec)

        def fsel():
            for l in range(L):
                sb, ns, mg, kp, wl = sels[l]
                D.select(qs[l], layers[l], budget, out=(sb, ns, mg, kp, wl, None), ws=ws_sel)

        def fused():  # the step as bench.py runs it: dynsplit_select (a5+a6), then a7, per layer
            for l in range(L):
                sb, ns, mg, kp, wl = sels[l]
                D.select(qs[l], layers[l], budget, out=(sb, ns, mg, kp, wl, None), ws=ws_sel)
                D.decode_attn(qs[l], layers[l], sels[l][4], out=outs[l], ws=ws_dec)

        ws_lay = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dev, "layer")

        def layer_api():  # dynsplit_decode_layer per layer
            for l in range(L):
                _, ns, mg, kp, wl = sels[l]
                D.decode_layer(qs[l], layers[l], budget, out=(ns, mg, kp, wl, outs[l][0], outs[l][1]),
                               ws=ws_lay)

        t_s, t_f, t_a, t_all, t_fs, t_fu, t_ly = (time_graph(f) / L for f in (score, selfs, attn, full, fsel,
                                                                              fused, layer_api))
        rows = sum(int(D.worklist_rows(sels[l][4], shape, Hq // Hkv)[1].sum()) for l in range(L)) / L
        mbytes = rows * 2 * d * 2 / 2**20
        print(f"budget {budget:6d}: score {t_s:5.1f} | select {t_f:5.1f} | select() {t_fs:5.1f} | attn {t_a:5.1f} us "
              f"({mbytes:6.1f} MiB, {mbytes * 2**20 / (t_a * 1e-6) / 1e9:5.0f} GB/s) | layer: 3-kernel {t_all:5.1f} "
              f"select()+attn {t_fu:5.1f} | decode_layer {t_ly:5.1f} us")

if __name__ == "__main__":
    main()

"""Prefill block construction stages (not part of the product) at the C5
shape: B sequences, 32Q/8KV, d = 128, bf16, one scored layer.
    python tools/exp_prefill_build.py [S] [B]
Times a1 (delimiter scoring), a2 (weight table), a3 (DD-Select), a4 (page
map; repack + digests) separately with CUDA events (each after a warm-up)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D  # noqa: E402
from synth import generators as G  # noqa: E402

dev = torch.device("cuda:0")
S = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
Hq, Hkv, d = 32, 8, 128
cfg = D.default_config()
toks = torch.from_numpy(np.stack([G.tokens(b, S) for b in range(B)])).to(dev)
ids = torch.from_numpy(G.T7_IDS).to(dev)
gen = torch.Generator(device=dev)
gen.manual_seed(2)
Qs = torch.randn(1, B, S, Hq, d, generator=gen, device=dev).to(torch.bfloat16)
Ks = torch.randn(1, B, S, Hkv, d, generator=gen, device=dev).to(torch.bfloat16)
K = torch.randn(B, S, Hkv, d, generator=gen, device=dev).to(torch.bfloat16)
V = torch.randn(B, S, Hkv, d, generator=gen, device=dev).to(torch.bfloat16)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


t1, s = timed(lambda: D.score_delimiters(toks, ids, Qs, Ks, cfg))
t2, w10 = timed(lambda: D.weight_table(toks, ids, s))
t3, (bs, nb) = timed(lambda: D.segment(toks, ids, w10, cfg))
t4a, (pf, pb, pv, npg) = timed(lambda: D.map_pages(bs, nb, S, cfg))
# outputs preallocated once: an allocation inside the timed loop (cudaMalloc of
# ~2.5 GiB at 128K, B = 4) would be timed as kernel time
kvd = D.repack_digest(K, V, bs, nb, pf, cfg)
t4b, _ = timed(lambda: D.repack_digest(K, V, bs, nb, pf, cfg, out=kvd))
rows = np.arange(S, dtype=np.float64) + 1
flop = 2.0 * d * Hq * rows.sum() * B
bytes4 = 2 * 2 * B * S * Hkv * d * 2 + int(nb.sum()) * Hkv * 2 * d * 2
print(f"C5 prefill, S={S}, B={B}, 32Q/8KV: a1 {t1:.2f} ms ({flop / (t1 * 1e-3) / 1e12:.0f} TFLOP/s) | "
      f"a2 {t2 * 1e3:.1f} us | a3 {t3 * 1e3:.1f} us | a4 map {t4a * 1e3:.1f} us, repack+digest {t4b * 1e3:.1f} us "
      f"({bytes4 / (t4b * 1e-3) / 1e9:.0f} GB/s) | blocks/seq {int(nb[0])}")

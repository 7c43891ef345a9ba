"""Seeded random shapes through dynsplit_decode_layer: the fused layer against
the three-kernel path (identical selections, worklists, o and lse) and the
oracle (selection exact on margin-certified queries, attention within R17),
plus the offloaded layer against the resident one.  Shapes, budgets, page
sizes and head layouts are drawn from a fixed generator, so a failure names
its case and reproduces exactly."""
import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G
from tests import helpers as H
from tests.test_gpu_fused import D, assert_same, build, check_oracle, run_both, t  # noqa: F401

pytestmark = pytest.mark.gpu

LAYOUTS = [(8, 8), (16, 8), (32, 8), (16, 2), (32, 4), (8, 1), (64, 8)]


def _cases(n=14, seed=424242, long=False):
    r = G.rng(seed, 1)
    out = []
    for i in range(n):
        Hq, Hkv = LAYOUTS[int(r.integers(len(LAYOUTS)))]
        B = int(r.integers(1, 4))
        S = int(r.choice([int(r.integers(1, 64)), int(r.integers(64, 4000)), int(r.integers(4000, 24000))]))
        if long:
            S = int(r.integers(24000, 140000))
            B = int(r.integers(1, 3))
        budget = int(r.choice([1, int(r.integers(2, 64)), int(r.integers(64, 2048)), S + 7]))
        P = int(r.choice([8, 16, 32]))
        out.append((i, B, S, Hq, Hkv, budget, P))
    return out


@pytest.mark.parametrize("case", _cases() + [(100 + c[0],) + c[1:] for c in _cases(6, 777, long=True)],
                         ids=lambda c: "c%d_B%d_S%d_H%d-%d_b%d_P%d" % c)
def test_fuzz_fused_vs_three_kernels_vs_oracle(D, case):
    i, B, S, Hq, Hkv, budget, P = case
    d = 128
    cfg = D.default_config(page_size=P)
    toks = np.stack([G.tokens(5000 + 10 * i + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, cfg.C, cfg.delta) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(5500 + 10 * i + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    q = H.certify_queries(5500 + 10 * i, q, K, starts, budget, "bf16")
    layer = build(D, toks, K, V, Hq, cfg)
    qt = t(q, torch.bfloat16)
    a, b = run_both(D, qt, layer, budget)
    assert_same(D, a, b, D.make_shape(B, S, Hq, Hkv, d), Hq // Hkv)
    check_oracle(a[2], a[0], a[1], H.oracle_decode(q, K, V, starts, budget), B, Hq)


@pytest.mark.parametrize("case", _cases(6), ids=lambda c: "c%d_B%d_S%d_H%d-%d_b%d_P%d" % c)
def test_fuzz_offload_equals_resident(D, case):
    """Two steps of the offloaded layer (cache empty, then reuse) give the
    resident path's o and lse on the same worklist, bit for bit."""
    i, B, S, Hq, Hkv, budget, P = case
    d = 128
    cfg = D.default_config(page_size=P)
    toks = np.stack([G.tokens(6000 + 10 * i + b, S) for b in range(B)])
    qs, Ks, Vs = zip(*[G.decode_qkv(6500 + 10 * i + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    layer = build(D, toks, K, V, Hq, cfg)
    off = D.offload_layer(layer, budget, Hq, keep_device=True)
    walk = G.decode_query_walk(6600 + i, 2, q, 0.9)
    for step in range(2):
        qt = t(walk[step], torch.bfloat16)
        o, lse, sel = D.decode_layer_offload(qt, off, budget)
        o_r, lse_r = D.decode_attn(qt, layer, sel.worklist)
        torch.cuda.synchronize()
        assert torch.equal(o, o_r) and torch.equal(lse, lse_r), step

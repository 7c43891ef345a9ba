"""The fused decode layer (k_decode_fused: a5 + a6 + a7 + a8 in one kernel)
against the three-kernel path (k_score_blocks_tc -> k_select_reg ->
k_decode_attn) and the oracle.

Both paths run behind dynsplit_decode_layer; dynsplit_debug_fused(0/1)
switches between them and dynsplit_debug_fused_launches() proves the fused
kernel actually ran.  The fused kernel must give bit-identical selections,
worklists, o and lse (same page assignment, same arithmetic), so every case
compares with torch.equal, then with the oracle (selection exact, attention
within DESIGN R17).  Cases cover the band fast path (continuous scores, also
skewed by outlier tails and at budget / total = 1/3: the local brackets of
R25 hold for any distribution), the
exact slow path (integer scores: massive ties; all-zero scores), all-fit
budgets, budget 1, G = 1 / 2 / 4 / 8, several sequences per launch, a plan
whose blocks are shorter than any DD-Select plan, and the digest staging in
several rounds (more blocks per CTA than one stage holds).
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G
from tests import helpers as H

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
ATT_TOL = 2e-3
LSE_TOL = 1e-4


@pytest.fixture(scope="module")
def D():
    from paper_2602_03184_b200 import dynsplit
    lib = dynsplit.lib()
    lib.dynsplit_debug_fused_launches.restype = ctypes.c_longlong
    yield dynsplit
    lib.dynsplit_debug_fused(1)


def t(x, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(x)).to(DEV, dtype=dtype)


def run_both(D, qt, layer, budget):
    """decode_layer through the fused kernel, then through the three kernels;
    returns both result sets (o, lse, n_sel, marginal, keep, worklist)."""
    lib = D.lib()
    outs = []
    for fused in (1, 0):
        lib.dynsplit_debug_fused(fused)
        before = lib.dynsplit_debug_fused_launches()
        o, lse, sel = D.decode_layer(qt, layer, budget)
        torch.cuda.synchronize()
        ran = lib.dynsplit_debug_fused_launches() - before
        assert ran == (1 if fused else 0), f"fused={fused}: {ran} fused launches"
        outs.append((o, lse, sel))
    lib.dynsplit_debug_fused(1)
    return outs


def assert_same(D, a, b, shape, G_):
    (o1, l1, s1), (o2, l2, s2) = a, b
    assert torch.equal(o1, o2), (o1 - o2).abs().max()
    assert torch.equal(l1, l2)
    for name in ("n_sel", "marginal_block", "marginal_keep"):
        assert torch.equal(getattr(s1, name), getattr(s2, name)), name
    # the worklists: same page entries in the same order for every (b, KV head)
    assert np.array_equal(worklist_entries(s1.worklist, shape), worklist_entries(s2.worklist, shape))


def worklist_entries(wl, shape):
    """Used entries {page, block, rows[8]} per (b, KV head), in order
    (layout: dynsplit.worklist_rows)."""
    raw = wl.cpu().numpy()
    nbh = shape.B * shape.Hkv
    max_wl = int(raw[:256].view(np.int32)[1])
    counts = raw[256:256 + 4 * nbh].view(np.int32)
    off = 256 + ((4 * nbh + 255) // 256) * 256
    ent = raw[off: off + 16 * nbh * max_wl].reshape(max_wl, nbh, 16).transpose(1, 0, 2)
    return np.concatenate([counts.astype(np.int64)] +
                          [ent[i, : counts[i]].reshape(-1).astype(np.int64) for i in range(nbh)])


def check_oracle(sel, o, lse, res, B, Hq):
    mg = sel.marginal_block.cpu().numpy()
    kp = sel.marginal_keep.cpu().numpy()
    ns = sel.n_sel.cpu().numpy()
    o = o.cpu().numpy()
    lse = lse.cpu().numpy()
    for b in range(B):
        r = res[b]
        for h in range(Hq):
            assert ns[b, h] == len(r["sel_blocks"][h]), (b, h)
            assert mg[b, h] == r["marginal"][h] and kp[b, h] == r["keep"][h], (b, h)
        assert np.all(H.row_rel_err(o[b], r["o"]) <= ATT_TOL)
        assert np.all(np.abs(lse[b] - r["lse"]) <= LSE_TOL * np.maximum(1, np.abs(r["lse"])))


def build(D, toks, K, V, Hq, cfg=None):
    cfg = cfg or D.default_config()
    return D.build_blocks(t(toks), t(G.T7_IDS), t(K, torch.bfloat16), t(V, torch.bfloat16), cfg,
                          static_w10=G.T7_W10, Hq=Hq)


@pytest.mark.parametrize("B,S,Hq,Hkv,budget,kind", [
    (1, 20000, 32, 8, 1024, "cont"),     # band fast path, G = 4
    (2, 9000, 16, 8, 700, "cont"),       # G = 2
    (1, 6000, 8, 8, 300, "cont"),        # G = 1 (MHA)
    (1, 8000, 32, 4, 500, "cont"),       # G = 8
    (3, 5000, 32, 8, 600, "int"),        # integer scores: ties -> slow path / equal keys
    (1, 4000, 32, 8, 1, "cont"),         # budget 1
    (2, 3000, 32, 8, 5000, "cont"),      # budget >= S: everything fits
    (1, 3000, 32, 8, 400, "zero"),       # q = 0: all scores equal (index order)
    (4, 2500, 32, 8, 256, "cont"),       # several sequences, few splits each
    (1, 20000, 32, 8, 1024, "lowtail"),  # a tail of low-score outlier blocks (skewed distribution)
    (1, 20000, 32, 8, 1024, "hightail"),  # a tail of high-score blocks, all in the last ranges
    (1, 12000, 32, 8, 4000, "cont"),     # budget / total = 1/3 (a wide crossing band)
])
def test_fused_equals_three_kernels_and_oracle(D, B, S, Hq, Hkv, budget, kind):
    d = 128
    toks = np.stack([G.tokens(3100 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    gen = G.decode_qkv_integer if kind == "int" else G.decode_qkv
    qs, Ks, Vs = zip(*[gen(3200 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    if kind == "lowtail":   # x 1/16 and x 4 keep the keys bf16-exact
        K[:, S - 1500:] *= 0.0625
    if kind == "hightail":
        K[:, S - 600:] *= 4.0
    if kind in ("cont", "lowtail", "hightail"):
        q = H.certify_queries(3200, q, K, starts, budget, "bf16")
    if kind == "zero":
        q = np.zeros_like(q)
    layer = build(D, toks, K, V, Hq)
    qt = t(q, torch.bfloat16)
    a, b = run_both(D, qt, layer, budget)
    shape = D.make_shape(B, S, Hq, Hkv, d)
    assert_same(D, a, b, shape, Hq // Hkv)
    if kind != "zero":
        res = H.oracle_decode(q, K, V, starts, budget)
        check_oracle(a[2], a[0], a[1], res, B, Hq)


@pytest.mark.parametrize("force", [1, 2])
@pytest.mark.parametrize("B,S,Hq,Hkv,budget,kind", [
    (1, 20000, 32, 8, 1024, "cont"),
    (1, 8000, 32, 4, 500, "lowtail"),    # G = 8
    (2, 9000, 16, 8, 700, "hightail"),
    (1, 6000, 8, 8, 300, "cont"),        # G = 1
    (1, 5000, 32, 8, 600, "int"),        # ties: the fallback's crossing bin overflows -> slow path
])
def test_fused_selection_paths(D, force, B, S, Hq, Hkv, budget, kind):
    """Every head forced through the histogram fallback (force = 1: the
    crossing bin of a kH-bin histogram over [gmin, gmax], R25) or through the
    CTA-wide slow path (force = 2): the same selections, worklists, o and lse
    as the three-kernel path, and the oracle's."""
    lib = D.lib()
    d = 128
    toks = np.stack([G.tokens(3500 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    gen = G.decode_qkv_integer if kind == "int" else G.decode_qkv
    qs, Ks, Vs = zip(*[gen(3600 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    if kind == "lowtail":
        K[:, S - 1500:] *= 0.0625
    if kind == "hightail":
        K[:, S - 600:] *= 4.0
    if kind != "int":
        q = H.certify_queries(3600, q, K, starts, budget, "bf16")
    layer = build(D, toks, K, V, Hq)
    qt = t(q, torch.bfloat16)
    lib.dynsplit_debug_fused_force(force)
    try:
        a, b = run_both(D, qt, layer, budget)
    finally:
        lib.dynsplit_debug_fused_force(0)
    assert_same(D, a, b, D.make_shape(B, S, Hq, Hkv, d), Hq // Hkv)
    res = H.oracle_decode(q, K, V, starts, budget)
    check_oracle(a[2], a[0], a[1], res, B, Hq)


def test_fused_staging_rounds_and_short_blocks(D):
    """A plan of 18-token blocks (the shortest non-final DD-Select length at
    C = 32, Delta = 14): more blocks per CTA than the launch hint sized the
    digest stage for, so phase 1 stages its range in several TMA rounds."""
    B, S, Hq, Hkv, d, budget = 1, 60000, 32, 8, 128, 2048
    toks = G.tokens(3300, S)[None]
    starts = list(range(0, S, 18)) + [S]
    qs, Ks, Vs = G.decode_qkv(3301, S, Hq, Hkv, d)
    q, K, V = qs[None], Ks[None], Vs[None]
    q = H.certify_queries(3301, q, K, [starts], budget, "bf16")
    cfg = D.default_config()
    base = build(D, toks, K, V, Hq, cfg)
    bs = torch.full((B, D.max_blocks(S, cfg) + 1), S, dtype=torch.int32)
    bs[:, : len(starts)] = torch.tensor(starts, dtype=torch.int32)
    bs = bs.to(DEV)
    nb = torch.full((B,), len(starts) - 1, dtype=torch.int32, device=DEV)
    pf, pb, pv, npg = D.map_pages(bs, nb, S, cfg)
    Kp, Vp, dig = D.repack_digest(t(K, torch.bfloat16), t(V, torch.bfloat16), bs, nb, pf, cfg)
    layer = D.PagedLayer(base.shape, cfg, base.w10, bs, nb, pf, pb, pv, npg, Kp, Vp, dig)
    qt = t(q, torch.bfloat16)
    a, b = run_both(D, qt, layer, budget)
    assert_same(D, a, b, D.make_shape(B, S, Hq, Hkv, d), Hq // Hkv)
    res = H.oracle_decode(q, K, V, [starts], budget)
    check_oracle(a[2], a[0], a[1], res, B, Hq)


def test_fused_layers_graph_replay(D):
    """Eight layers back to back on one workspace (the group barriers and the
    split tickets are reused across launches), captured in a CUDA graph and
    replayed three times: every replay equals the eager result bit for bit."""
    B, S, Hq, Hkv, d, budget, L = 1, 12000, 32, 8, 128, 800, 8
    toks = G.tokens(3400, S)[None]
    layers, qts = [], []
    for l in range(L):
        q, K, V = G.decode_qkv(3410 + l, S, Hq, Hkv, d)
        layers.append(build(D, toks, K[None], V[None], Hq))
        qts.append(t(q[None], torch.bfloat16))
    shape = D.make_shape(B, S, Hq, Hkv, d)
    cfg = layers[0].cfg
    ws = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), DEV, "fused_graph")
    outs = [(torch.empty(B, Hq, d, device=DEV), torch.empty(B, Hq, device=DEV)) for _ in range(L)]
    sel = D._sel_outputs(shape, cfg, budget, DEV, want_blocks=False)

    def step():
        for l in range(L):
            _, ns, mg, kp, wl = sel
            D.decode_layer(qts[l], layers[l], budget, out=(ns, mg, kp, wl, outs[l][0], outs[l][1]), ws=ws)

    step()
    torch.cuda.synchronize()
    ref = [(o.clone(), l.clone()) for o, l in outs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        for o, l in outs:
            o.zero_()
            l.zero_()
        g.replay()
        torch.cuda.synchronize()
        for (o, l), (ro, rl) in zip(outs, ref):
            assert torch.equal(o, ro) and torch.equal(l, rl)
    assert D.read_device_error(ws) == 0


def test_step_host_layers_equals_device_layers(D):
    """dynsplit_decode_step_host_layers (one H2D of every layer's q, the
    layers back to back, one D2H each of o and lse) equals dynsplit_decode_layer
    per layer bit for bit."""
    B, S, Hq, Hkv, d, budget, L = 2, 6000, 32, 8, 128, 500, 3
    toks = np.stack([G.tokens(3500 + b, S) for b in range(B)])
    layers, qs = [], []
    for l in range(L):
        q, K, V = zip(*[G.decode_qkv(3510 + 10 * l + b, S, Hq, Hkv, d) for b in range(B)])
        layers.append(build(D, toks, np.stack(K), np.stack(V), Hq))
        qs.append(t(np.stack(q), torch.bfloat16))
    ref = [D.decode_layer(qs[l], layers[l], budget)[:2] for l in range(L)]
    q_h = torch.stack([x.cpu() for x in qs]).pin_memory()
    o_h = torch.empty(L, B, Hq, d).pin_memory()
    l_h = torch.empty(L, B, Hq).pin_memory()
    shape = D.make_shape(B, S, Hq, Hkv, d)
    ws = D.workspace(D.step_host_layers_workspace_bytes(shape, layers[0].cfg, budget, L), DEV, "shl_test")
    wl = D._sel_outputs(shape, layers[0].cfg, budget, DEV, want_blocks=False)[4]
    D.decode_step_host_layers(q_h, layers, budget, o_h, l_h, wl, ws)
    torch.cuda.synchronize()
    for l in range(L):
        assert torch.equal(o_h[l], ref[l][0].cpu()) and torch.equal(l_h[l], ref[l][1].cpu())


# ---------------------------------------------------------------- NEXT-2 variants (DESIGN R23, R24)
@pytest.mark.parametrize("gqa,whole,kind", [(1, 0, "int"), (1, 0, "cont"), (0, 1, "cont"), (0, 1, "int"),
                                            (1, 1, "cont")])
def test_fused_variants_against_oracle(D, gqa, whole, kind):
    """Group-shared GQA selection and the whole-block budget through
    dynsplit_decode_layer (fused), against oracle.decode_step(gqa_mode,
    budget_mode): selections exact, attention within R17; group mode streams
    exactly the budget per (sequence, KV head) (the union is 1x)."""
    B, S, Hq, Hkv, d, budget = 2, 9000, 32, 8, 128, 700
    toks = np.stack([G.tokens(3600 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    gen = G.decode_qkv_integer if kind == "int" else G.decode_qkv
    qs, Ks, Vs = zip(*[gen(3700 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    if kind == "lowtail":   # x 1/16 and x 4 keep the keys bf16-exact
        K[:, S - 1500:] *= 0.0625
    if kind == "hightail":
        K[:, S - 600:] *= 4.0
    if kind in ("cont", "lowtail", "hightail"):
        q = (H.certify_queries_group(3700, q, K, starts, budget) if gqa
             else H.certify_queries(3700, q, K, starts, budget, "bf16"))
    cfg = D.default_config(gqa_mode=gqa, budget_mode=whole)
    layer = D.build_blocks(t(toks), t(G.T7_IDS), t(K, torch.bfloat16), t(V, torch.bfloat16), cfg,
                           static_w10=G.T7_W10, Hq=Hq)
    qt = t(q, torch.bfloat16)
    o, lse, sel = D.decode_layer(qt, layer, budget)
    torch.cuda.synchronize()
    res = [O.decode_step(q[b], K[b], V[b], starts[b], budget, gqa_mode="group" if gqa else "head",
                         budget_mode="whole" if whole else "token") for b in range(B)]
    check_oracle(sel, o, lse, res, B, Hq)
    if gqa and not whole:
        shape = D.make_shape(B, S, Hq, Hkv, d)
        _, streamed = D.worklist_rows(sel.worklist, shape, Hq // Hkv)
        assert np.all(streamed == budget), streamed


def test_variants_unsupported_outside_the_fused_layer(D):
    """The NEXT-2 variants exist only in the fused layer: dynsplit_select
    refuses them (UNSUPPORTED) instead of silently selecting per head."""
    S, Hq, Hkv, d = 3000, 8, 2, 128
    toks = G.tokens(3800, S)[None]
    q, K, V = G.decode_qkv(3801, S, Hq, Hkv, d)
    cfg = D.default_config(gqa_mode=1)
    layer = D.build_blocks(t(toks), t(G.T7_IDS), t(K[None], torch.bfloat16), t(V[None], torch.bfloat16), cfg,
                           static_w10=G.T7_W10, Hq=Hq)
    with pytest.raises(D.DynsplitError):
        D.select(t(q[None], torch.bfloat16), layer, 300)


@pytest.mark.parametrize("B,S,Hq,Hkv,budget,kind", [
    (1, 20000, 32, 8, 1024, "cont"),
    (8, 3000, 32, 8, 300, "cont"),
    (3, 5000, 32, 8, 600, "int"),
    (1, 6000, 8, 8, 300, "hightail"),
    (2, 3000, 32, 8, 5000, "cont"),      # all fit
])
def test_fused_local_selection(D, monkeypatch, B, S, Hq, Hkv, budget, kind):
    """The local-selection mode (every CTA selects every head from the full
    score rows right after barrier A; the default for short sequences over
    few splits), forced on: the same selections, worklists, o and lse as the
    three kernels, and the oracle's."""
    monkeypatch.setenv("DYNSPLIT_FUSED_LOCAL", "1")
    d = 128
    toks = np.stack([G.tokens(3600 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    gen = G.decode_qkv_integer if kind == "int" else G.decode_qkv
    qs, Ks, Vs = zip(*[gen(3700 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    if kind == "hightail":
        K[:, S - 600:] *= 4.0
    if kind != "int":
        q = H.certify_queries(3700, q, K, starts, budget, "bf16")
    layer = build(D, toks, K, V, Hq)
    a, b = run_both(D, t(q, torch.bfloat16), layer, budget)
    assert_same(D, a, b, D.make_shape(B, S, Hq, Hkv, d), Hq // Hkv)
    check_oracle(a[2], a[0], a[1], H.oracle_decode(q, K, V, starts, budget), B, Hq)


def test_fused_adaptive_local_selection(D):
    """After a launch whose moment bounds missed (forced here through the
    test hook), the group's next launches select locally (a countdown in the
    group's barrier word 1, sequences of <= ~2600 blocks): the countdown is
    set to 8 and then decrements, and every launch equals the three-kernel
    path."""
    lib = D.lib()
    B, S, Hq, Hkv, d, budget = 1, 20000, 32, 8, 128, 1024
    toks = G.tokens(3900, S)[None]
    q, K, V = G.decode_qkv(3901, S, Hq, Hkv, d)
    starts = [O.segment(toks[0], G.T7_IDS, G.T7_W10, 32, 14)]
    q = H.certify_queries(3901, q[None], K[None], starts, budget, "bf16")
    layer = build(D, toks, K[None], V[None], Hq)
    qt = t(q, torch.bfloat16)
    shape = D.make_shape(B, S, Hq, Hkv, d)
    ws = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, shape, layer.cfg, budget), DEV, "adaptive_test")
    ws.zero_()
    # the group barrier words: workspace header (256 B), then the decode
    # body's counters (65536 int32), the barriers in their upper half,
    # 8 + 64 words per (b, KV head)
    words = ws[256:256 + 65536 * 4].view(torch.int32)[32768:]

    def state():
        torch.cuda.synchronize()
        return [int(words[bh * 72 + 1]) for bh in range(B * Hkv)]

    ref_o, ref_l, _ = D.decode_layer(qt, layer, budget, ws=ws)
    assert state() == [0] * (B * Hkv)
    lib.dynsplit_debug_fused_force(1)          # every head through the exact fallback: a "miss"
    try:
        o1, l1, _ = D.decode_layer(qt, layer, budget, ws=ws)
    finally:
        lib.dynsplit_debug_fused_force(0)
    assert state() == [8] * (B * Hkv)
    for k in range(3):                          # local selection, counting down
        o2, l2, _ = D.decode_layer(qt, layer, budget, ws=ws)
        assert state() == [7 - k] * (B * Hkv)
        assert torch.equal(o2, ref_o) and torch.equal(l2, ref_l)
    assert torch.equal(o1, ref_o) and torch.equal(l1, ref_l)
    res = H.oracle_decode(q, K[None], V[None], starts, budget)
    assert np.all(H.row_rel_err(o2[0].cpu().numpy(), res[0]["o"]) <= ATT_TOL)

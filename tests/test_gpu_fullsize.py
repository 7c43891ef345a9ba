"""Full-size parity at BASELINE.json's sizes, in the launch configuration
bench.py times (dynsplit_decode_layer, same grids): config 3 per-GPU shard
(128K, 32Q/8KV, budget 4096, bf16), config 4 heads (40 MHA) at 128K, config 2
(32K, budget 2K) and the config 5 prefill scoring at 64K on sampled
candidates.

Outputs the oracle can compute directly (plans, page maps, every head's
selection and attention output) are compared in full; digests and delimiter
scores on samples."""
import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G
from tests import helpers as H

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda:0"


def t(x, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(x)).to(DEV, dtype=dtype)


@pytest.mark.parametrize("S,Hq,Hkv,budget", [(131072, 32, 8, 4096), (131072, 40, 40, 4096),
                                             (32768, 32, 8, 2048)])
def test_decode_128k(S, Hq, Hkv, budget):
    """Configs 3 (per-GPU shard), 4 (40 MHA heads) and 2 (32K, budget 2K)."""
    from paper_2602_03184_b200 import dynsplit as D
    d = 128
    cfg = D.default_config()
    toks = G.tokens(2000, S)
    q, K, V = G.decode_qkv(2001, S, Hq, Hkv, d)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, cfg.C, cfg.delta)
    q = H.certify_queries(2001, q[None], K[None], [starts], budget)[0]
    layer = D.build_blocks(t(toks[None]), t(G.T7_IDS), t(K[None], torch.bfloat16),
                           t(V[None], torch.bfloat16), cfg, static_w10=G.T7_W10, Hq=Hq)
    qt = t(q[None], torch.bfloat16)
    sel = D.select(qt, layer, budget)
    o, lse = D.decode_attn(qt, layer, sel.worklist)
    o_d, lse_d = D.decode_attn(qt, layer, None)
    o_l, lse_l, sel_l = D.decode_layer(qt, layer, budget)   # the call bench.py times
    torch.cuda.synchronize()
    assert torch.equal(o_l, o) and torch.equal(lse_l, lse) and torch.equal(sel_l.n_sel, sel.n_sel)
    nb = int(layer.n_blocks[0])
    assert layer.block_starts[0, : nb + 1].tolist() == starts
    pf, pb, pv = O.page_map(starts, cfg.page_size)
    assert layer.page_first[0, : nb + 1].tolist() == pf.tolist()
    assert layer.page_valid[0, : int(pf[-1])].tolist() == pv.tolist()
    kmax, kmin = O.digests(K, starts)
    r = G.rng(5, 6)
    sample = r.choice(nb, size=64, replace=False)
    dig = layer.digests[0].float().cpu().numpy()
    assert np.array_equal(dig[:, sample, 0], kmax[:, sample]) and np.array_equal(dig[:, sample, 1], kmin[:, sample])
    res = O.decode_step(q, K, V, starts, budget)
    ns = sel.n_sel.cpu().numpy()[0]
    sb = sel.sel_blocks.cpu().numpy()[0]
    for h in range(Hq):
        assert sb[h, : ns[h]].tolist() == res["sel_blocks"][h], h
        assert int(sel.marginal_block[0, h]) == res["marginal"][h]
        assert int(sel.marginal_keep[0, h]) == res["keep"][h]
    err = H.row_rel_err(o[0].cpu().numpy(), res["o"])
    assert np.all(err <= 2e-3), err.max()
    assert np.all(np.abs(lse[0].cpu().numpy() - res["lse"]) <= 1e-4 * np.maximum(1, np.abs(res["lse"])))
    g = Hq // Hkv
    for h in (0, Hq - 1):                               # dense baseline on two heads
        od, ld = O.dense_attention(q[h], K[:, h // g], V[:, h // g], 1 / np.sqrt(d))
        assert H.row_rel_err(o_d[0, h].cpu().numpy()[None], od[None])[0] <= 2e-3
        assert abs(float(lse_d[0, h]) - ld) <= 1e-4 * max(1, abs(ld))


def test_prefill_scoring_64k_sampled():
    from paper_2602_03184_b200 import dynsplit as D
    S, Hq, Hkv, d = 65536, 32, 8, 128
    cfg = D.default_config()
    toks = G.tokens(2100, S)
    Qs, Ks = G.scoring_qk(2101, 1, S, Hq, Hkv, d)
    s = D.score_delimiters(t(toks[None]), t(G.T7_IDS), t(Qs[:, None], torch.bfloat16),
                           t(Ks[:, None], torch.bfloat16), cfg).cpu().numpy()[0]
    dset = set(G.T7_IDS.tolist())
    cands = np.array([i for i in range(S - 1) if int(toks[i]) in dset])
    r = G.rng(7, 8)
    sample = np.concatenate([cands[:4], cands[-4:], r.choice(cands, size=8, replace=False)])
    ref = O.score_delimiters(toks, G.T7_IDS, Qs, Ks, cfg.W, cfg.R, cfg.alpha_pen, candidates=sample.tolist())
    for i in sample:
        assert abs(s[i] - ref[i]) <= 2e-4, (i, s[i], ref[i])
    assert np.isnan(s[S - 1]) and np.sum(~np.isnan(s)) == len(cands)


def test_decode_128k_batch8():
    """Config 3 unsharded (all 8 sequences of 128K on one GPU, the bench's
    c3_b8 block) through dynsplit_decode_layer, every head of every sequence
    against the oracle.  At this shape the fused layer declines (2 splits per
    (sequence, KV head): a range's scores do not fit one SM's shared memory;
    a variant re-staging them in region A measured 143 vs 132 us per layer,
    DESIGN section 8) and the layer runs the three kernels, which must equal
    dynsplit_select + dynsplit_decode_attn bit for bit."""
    from paper_2602_03184_b200 import dynsplit as D
    B, S, Hq, Hkv, d, budget = 8, 131072, 32, 8, 128, 4096
    cfg = D.default_config()
    toks = np.stack([G.tokens(2200 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, cfg.C, cfg.delta) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(2300 + b, S, Hq, Hkv, d) for b in range(B)])
    q = np.stack(qs)
    q = H.certify_queries(2300, q, np.stack(Ks), starts, budget)
    layer = D.build_blocks(t(toks), t(G.T7_IDS), t(np.stack(Ks), torch.bfloat16), t(np.stack(Vs), torch.bfloat16),
                           cfg, static_w10=G.T7_W10, Hq=Hq)
    qt = t(q, torch.bfloat16)
    import ctypes
    lib = D.lib()
    lib.dynsplit_debug_fused_launches.restype = ctypes.c_longlong
    n0 = lib.dynsplit_debug_fused_launches()
    o_l, lse_l, sel_l = D.decode_layer(qt, layer, budget)
    assert lib.dynsplit_debug_fused_launches() - n0 == 0          # three kernels at this shape
    sel = D.select(qt, layer, budget)
    o, lse = D.decode_attn(qt, layer, sel.worklist)
    torch.cuda.synchronize()
    assert torch.equal(o_l, o) and torch.equal(lse_l, lse)
    for name in ("n_sel", "marginal_block", "marginal_keep"):
        assert torch.equal(getattr(sel_l, name), getattr(sel, name)), name
    o_np, lse_np = o_l.cpu().numpy(), lse_l.cpu().numpy()
    mg, kp, ns = sel_l.marginal_block.cpu().numpy(), sel_l.marginal_keep.cpu().numpy(), sel_l.n_sel.cpu().numpy()
    for b in range(B):
        res = O.decode_step(q[b], Ks[b], Vs[b], starts[b], budget)
        for h in range(Hq):
            assert ns[b, h] == len(res["sel_blocks"][h]) and mg[b, h] == res["marginal"][h] \
                and kp[b, h] == res["keep"][h], (b, h)
        assert np.all(H.row_rel_err(o_np[b], res["o"]) <= 2e-3)
        assert np.all(np.abs(lse_np[b] - res["lse"]) <= 1e-4 * np.maximum(1, np.abs(res["lse"])))


def test_offload_reuse_32k():
    """NEXT-3 at config 2's size (32K, 32Q/8KV, budget 2K) with the page cache
    sized by dynsplit_cache_slots, through dynsplit_decode_layer_offload over a
    3-step query walk: every KV head's page set, moved (fresh) pages, reuse
    counts and reuse_len bit-exact against O.offload_decode_loop, o / lse
    bit-identical to the resident path and within R17 of the oracle."""
    from paper_2602_03184_b200 import dynsplit as D
    S, Hq, Hkv, d, budget, T = 32768, 32, 8, 128, 2048, 3
    cfg = D.default_config()
    toks = G.tokens(2100, S)
    q0, K, V = G.decode_qkv(2101, S, Hq, Hkv, d)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, cfg.C, cfg.delta)
    qs = G.decode_query_walk(2102, T, q0, 0.9)
    qs = np.stack([H.certify_queries(2103 + i, qs[i][None], K[None], [starts], budget)[0] for i in range(T)])
    layer = D.build_blocks(t(toks[None]), t(G.T7_IDS), t(K[None], torch.bfloat16),
                           t(V[None], torch.bfloat16), cfg, static_w10=G.T7_W10, Hq=Hq)
    off = D.offload_layer(layer, budget, Hq, keep_device=True)
    shape = D.make_shape(1, S, Hq, Hkv)
    ref = O.offload_decode_loop(qs, K, V, starts, budget, P=cfg.page_size, truncate=True)
    for i in range(T):
        qt = t(qs[i][None], torch.bfloat16)
        o, lse, sel = D.decode_layer_offload(qt, off, budget)
        o_r, lse_r = D.decode_attn(qt, layer, sel.worklist)
        torch.cuda.synchronize()
        assert torch.equal(o, o_r) and torch.equal(lse, lse_r)
        pages = D.worklist_pages(sel.worklist, shape)
        fc = off.fetch_count.cpu().numpy()[0]
        fl = off.fetch.cpu().numpy()[0]
        st = off.reuse_stats.cpu().numpy()[0]
        r = ref[i]
        for hk in range(Hkv):
            assert np.sort(pages[hk]).tolist() == r["pages"][hk].tolist(), (i, hk)
            assert fl[hk, : fc[hk], 0].tolist() == r["fresh"][hk].tolist(), (i, hk)
            assert st[hk].tolist() == [len(r["reused"][hk]), len(r["fresh"][hk])], (i, hk)
        assert int(off.reuse_len[0]) == r["reuse_len"]
        assert np.all(H.row_rel_err(o[0].cpu().numpy(), r["o"]) <= 2e-3)
        assert np.all(np.abs(lse[0].cpu().numpy() - r["lse"]) <= 1e-4 * np.maximum(1, np.abs(r["lse"])))
    assert sum(len(x) for x in ref[-1]["reused"]) > 0

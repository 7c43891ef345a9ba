"""Pins for oracle O5-O9: digests, block scores, budgeted
top-k via block-to-token mapping, attention over the
selection and the LSE merge."""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EX = json.load(open(os.path.join(GOLD, "v2f_examples.json")))


def test_digest_examples():
    ex = EX["digest_two_tokens"]
    K = np.array(ex["keys"], float)[:, None, :]
    kmax, kmin = O.digests(K, [0, 2])
    assert kmax[0, 0].tolist() == ex["key_max"] and kmin[0, 0].tolist() == ex["key_min"]
    kmax, kmin = O.digests(K, [0, 1, 2])          # singleton blocks
    assert np.array_equal(kmax[0], K[:, 0]) and np.array_equal(kmin[0], K[:, 0])


def test_digest_containment():
    _, K, _ = G.decode_qkv(1, 700, 4, 2, 32)
    starts = O.segment(G.tokens(1, 700), G.T7_IDS, G.T7_W10, 32, 14)
    kmax, kmin = O.digests(K, starts)
    for b in range(len(starts) - 1):
        blk = K[starts[b]:starts[b + 1]].transpose(1, 0, 2)   # [H, n, d]
        assert np.all(blk <= kmax[:, b, None, :]) and np.all(blk >= kmin[:, b, None, :])
        assert np.all(np.any(blk == kmax[:, b, None, :], axis=1))
        assert np.all(np.any(blk == kmin[:, b, None, :], axis=1))


def test_block_score_special_cases_and_upper_bound():
    q, K, _ = G.decode_qkv(2, 500, 4, 2, 32)
    starts = O.segment(G.tokens(2, 500), G.T7_IDS, G.T7_W10, 32, 14)
    kmax, kmin = O.digests(K, starts)
    for h in range(4):
        sc = O.block_scores(q[h], kmax[h // 2], kmin[h // 2])
        for b in range(len(starts) - 1):
            dots = K[starts[b]:starts[b + 1], h // 2, :].astype(np.float64) @ q[h].astype(np.float64)
            assert sc[b] >= dots.max() - 1e-9           # S:281 upper bound
    # singleton block -> exact q.k; zero query -> 0
    k1 = K[:1, 0, :]
    assert O.block_scores(q[0], k1, k1)[0] == pytest.approx(float(k1[0].astype(float) @ q[0].astype(float)), abs=1e-12)
    assert np.all(O.block_scores(np.zeros(32), kmax[0], kmin[0]) == 0)


@pytest.mark.parametrize("name", ["select_tie", "map_block_to_tokens"])
def test_selection_examples(name):
    ex = EX[name]
    toks = O.select_tokens(ex["scores"], ex["block_starts"], ex["budget"])
    sb, m, keep = O.selection_from_tokens(toks, ex["scores"], ex["block_starts"], ex["budget"])
    assert (sb, m, keep) == (ex["sel_blocks"], ex["marginal"], ex["keep"])
    if "tokens" in ex:
        assert toks.tolist() == ex["tokens"]


@pytest.mark.parametrize("seed", range(60))
def test_token_sort_equals_block_fill(seed):
    # S:301 / S:522: the materialised per-token stable sort equals an
    # independent block-order fill, including integer scores with many ties.
    r = G.rng(seed, 12)
    S = int(r.integers(1, 600))
    starts = O.segment(G.tokens(seed, S), G.T7_IDS, G.T7_W10, int(r.integers(4, 40)), 3)
    nb = len(starts) - 1
    scores = r.integers(-3, 4, size=nb).astype(float) if seed % 2 else r.standard_normal(nb)
    budget = int(r.integers(1, S + 20))
    toks = O.select_tokens(scores, starts, budget)
    sb, m, keep = O.selection_from_tokens(toks, scores, starts, budget)
    sb2, m2, keep2, toks2 = O.select_blocks_direct(scores, starts, budget)
    assert (sb, m, keep) == (sb2, m2, keep2)
    assert np.array_equal(toks, toks2)
    assert len(toks) == min(budget, S)             # budget exactness
    if budget >= S:
        assert m == -1 and len(toks) == S


def test_attention_matches_torch_sdpa():
    q, K, V = G.decode_qkv(3, 400, 8, 2, 64)
    scale = 1 / math.sqrt(64)
    for h in range(8):
        o, lse = O.dense_attention(q[h], K[:, h // 4], V[:, h // 4], scale)
        qt = torch.tensor(q[h], dtype=torch.float64)[None, None, None, :]
        kt = torch.tensor(K[:, h // 4], dtype=torch.float64)[None, None]
        vt = torch.tensor(V[:, h // 4], dtype=torch.float64)[None, None]
        ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, scale=scale)[0, 0, 0].numpy()
        assert np.allclose(o, ref, atol=1e-12)
        lse_ref = torch.logsumexp(torch.tensor(K[:, h // 4], dtype=torch.float64) @ torch.tensor(q[h], dtype=torch.float64) * scale, 0).item()
        assert lse == pytest.approx(lse_ref, abs=1e-12)


def test_sparse_attention_special_cases():
    q, K, V = G.decode_qkv(4, 300, 2, 1, 32)
    sc = 1 / math.sqrt(32)
    o, _ = O.sparse_attention(q[0], K[:, 0], V[:, 0], [17], sc)
    assert np.array_equal(o, V[17, 0].astype(np.float64))
    Keq = np.repeat(K[:1, 0], 300, axis=0)
    o, lse = O.dense_attention(q[0], Keq, V[:, 0], sc)
    assert np.allclose(o, V[:, 0].astype(np.float64).mean(0), atol=1e-12)
    with pytest.raises(ValueError):
        O.sparse_attention(q[0], K[:, 0], V[:, 0], [], sc)


def test_masked_dense_equivalence():
    # S:367 / S:402: attention over the selection equals dense attention with
    # non-selected logits set to -inf (library SDPA with a boolean mask).
    q, K, V = G.decode_qkv(5, 500, 4, 2, 64)
    starts = O.segment(G.tokens(5, 500), G.T7_IDS, G.T7_W10, 32, 14)
    res = O.decode_step(q, K, V, starts, 77)
    for h in range(4):
        mask = torch.zeros(1, 1, 1, 500, dtype=torch.bool)
        mask[..., torch.tensor(res["tokens"][h])] = True
        qt = torch.tensor(q[h], dtype=torch.float64)[None, None, None]
        kt = torch.tensor(K[:, h // 2], dtype=torch.float64)[None, None]
        vt = torch.tensor(V[:, h // 2], dtype=torch.float64)[None, None]
        ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask, scale=1 / 8)
        assert np.allclose(res["o"][h], ref[0, 0, 0].numpy(), atol=1e-12)
        assert len(res["tokens"][h]) == 77


def test_full_budget_equals_dense():
    q, K, V = G.decode_qkv(6, 256, 4, 4, 32)
    starts = O.segment(G.tokens(6, 256), G.T7_IDS, G.T7_W10, 32, 14)
    res = O.decode_step(q, K, V, starts, 10_000)
    for h in range(4):
        o, lse = O.dense_attention(q[h], K[:, h], V[:, h], 1 / math.sqrt(32))
        assert np.allclose(res["o"][h], o, atol=1e-12) and res["lse"][h] == pytest.approx(lse, abs=1e-12)
        assert res["marginal"][h] == -1


def test_merge_of_splits_equals_one_pass():
    q, K, V = G.decode_qkv(7, 333, 1, 1, 32)
    sc = 1 / math.sqrt(32)
    full_o, full_lse = O.dense_attention(q[0], K[:, 0], V[:, 0], sc)
    r = G.rng(7, 13)
    for _ in range(10):
        cuts = sorted(set(r.integers(1, 333, size=int(r.integers(1, 6))).tolist()))
        parts = np.split(np.arange(333), cuts)
        os_, ls_ = zip(*[O.sparse_attention(q[0], K[:, 0], V[:, 0], p, sc) for p in parts])
        # an empty part contributes lse = -inf
        o, L = O.merge_partials(np.vstack(os_ + (np.zeros(32),)), np.array(ls_ + (-np.inf,)))
        assert np.allclose(o, full_o, atol=1e-12) and L == pytest.approx(full_lse, abs=1e-12)
    o, L = O.merge_partials(np.zeros((2, 32)), np.array([-np.inf, -np.inf]))
    assert L == -np.inf and np.all(o == 0)


# ---------------------------------------------------------------- NEXT-2: mean-pooling digests
def test_mean_digest_special_cases():
    r = G.rng(31, 1)
    K = r.standard_normal((10, 2, 8))
    starts = [0, 1, 4, 10]
    km = O.digests_mean(K, starts)
    assert np.array_equal(km[:, 0, :], K[0])                       # singleton block -> k
    assert np.allclose(km[:, 1, :], (K[1] + K[2] + K[3]) / 3, rtol=0, atol=1e-15)
    Kc = np.ones((6, 1, 4)) * 2.5                                  # constant block -> the constant
    assert np.array_equal(O.digests_mean(Kc, [0, 6])[0, 0], np.full(4, 2.5))
    kmax, kmin = O.digests(K, starts)
    assert np.all(km <= kmax) and np.all(km >= kmin)               # containment


@pytest.mark.parametrize("seed", range(3))
def test_mean_score_is_mean_of_token_scores(seed):
    # linearity: q . mean_t(k_t) = mean_t (q . k_t), checked token by token
    r = G.rng(32, seed)
    S, d = 200, 16
    K = r.standard_normal((S, 1, d))
    q = r.standard_normal(d)
    starts = [0, 7, 40, 41, 90, 200]
    sc = O.block_scores_mean(q, O.digests_mean(K, starts)[0])
    for b in range(len(starts) - 1):
        toks = [float(np.dot(q, K[t, 0])) for t in range(starts[b], starts[b + 1])]
        assert abs(sc[b] - sum(toks) / len(toks)) <= 1e-12 * (1 + abs(sc[b]))


def test_mean_mode_full_budget_equals_dense():
    q, K, V = G.decode_qkv(33, 300, 4, 2, 16)
    starts = O.segment(G.tokens(33, 300), G.T7_IDS, G.T7_W10, 32, 14)
    res = O.decode_step(q, K, V, starts, 10_000, digest_mode="mean")
    for h in range(4):
        o, lse = O.dense_attention(q[h], K[:, h // 2], V[:, h // 2], 1 / math.sqrt(16))
        assert np.allclose(res["o"][h], o, rtol=0, atol=1e-12) and abs(res["lse"][h] - lse) < 1e-12


# ---------------------------------------------------------------- NEXT-2 variants (DESIGN R23, R24)
def _rand_plan(r, S, lo=18, hi=46):
    bs = [0]
    while bs[-1] < S:
        bs.append(min(S, bs[-1] + int(r.integers(lo, hi + 1))))
    return bs


@pytest.mark.parametrize("seed", range(6))
def test_group_scores_bound_the_group_logits(seed):
    """Sum of the heads' Quest bounds >= sum over heads of each head's best
    logit in the block >= the best summed logit of one token (an upper bound
    of the group's attention logits, brute force over tokens)."""
    r = G.rng(seed, 41)
    S, g, d = 300, 4, 16
    K = r.standard_normal((S, 1, d))
    q = r.standard_normal((g, d))
    bs = _rand_plan(r, S, 3, 12)
    kmax, kmin = O.digests(K, bs)
    sc = O.group_block_scores(q, kmax[0], kmin[0])
    for b in range(len(bs) - 1):
        logits = q @ K[bs[b]:bs[b + 1], 0].T          # [g, len]
        assert sc[b] >= logits.max(axis=1).sum() - 1e-9
        assert logits.max(axis=1).sum() >= logits.sum(axis=0).max() - 1e-9


def test_group_mode_reduces_to_per_head():
    """g = 1 (MHA): group mode is the per-head method; identical queries in a
    group: the group score is g x each head's score, so every head selects
    what per-head selection selects."""
    r = G.rng(3, 42)
    S, d = 400, 16
    bs = _rand_plan(r, S)
    K, V = r.standard_normal((S, 2, d)), r.standard_normal((S, 2, d))
    q1 = r.standard_normal((2, d))
    a = O.decode_step(q1, K, V, bs, 90, gqa_mode="group")
    b = O.decode_step(q1, K, V, bs, 90)
    assert a["sel_blocks"] == b["sel_blocks"] and a["marginal"] == b["marginal"] and a["keep"] == b["keep"]
    assert np.array_equal(a["o"], b["o"])
    q4 = np.repeat(r.standard_normal((2, 1, d)), 4, axis=1).reshape(8, d)   # Hq = 8, Hkv = 2, identical in-group
    a = O.decode_step(q4, K, V, bs, 90, gqa_mode="group")
    b = O.decode_step(q4, K, V, bs, 90)
    assert a["sel_blocks"] == b["sel_blocks"] and a["marginal"] == b["marginal"]


@pytest.mark.parametrize("seed", range(4))
def test_group_mode_shares_one_selection_of_exactly_budget(seed):
    """Every head of a KV group takes the same tokens, exactly `budget` of
    them, so the union over the group is 1x the budget."""
    r = G.rng(seed, 43)
    S, Hq, Hkv, d, budget = 600, 8, 2, 16, 150
    bs = _rand_plan(r, S)
    K, V = r.standard_normal((S, Hkv, d)), r.standard_normal((S, Hkv, d))
    q = r.standard_normal((Hq, d))
    res = O.decode_step(q, K, V, bs, budget, gqa_mode="group")
    for hk in range(Hkv):
        toks = [res["tokens"][h].tolist() for h in range(hk * 4, hk * 4 + 4)]
        assert all(t == toks[0] for t in toks) and len(toks[0]) == budget


@pytest.mark.parametrize("seed", range(8))
def test_whole_blocks_extend_the_token_selection(seed):
    """Whole-block budget = the token-exact selection plus the rest of its
    marginal block: >= budget tokens, fewer than budget + the marginal
    block's length, every selected block whole; a budget ending on a block
    boundary selects the same tokens in both modes; budget >= S takes all."""
    r = G.rng(seed, 44)
    S = 500
    bs = _rand_plan(r, S)
    sc = r.standard_normal(len(bs) - 1)
    sc[r.integers(0, len(sc), 5)] = sc[0]                      # ties
    for budget in (1, 37, 120, 499, 500, 900):
        blocks, m, ln, toks = O.select_whole_blocks(sc, bs, budget)
        exact = O.select_tokens(sc, bs, budget)
        if budget >= S:
            assert m == -1 and len(toks) == S
            continue
        sb, m2, keep = O.selection_from_tokens(exact, sc, bs, budget)
        assert blocks == sb and m == m2 and ln == bs[m + 1] - bs[m]
        assert set(exact.tolist()) <= set(toks.tolist())
        assert budget <= len(toks) < budget + ln
        assert len(toks) - len(exact) == ln - keep
        for b in blocks:
            assert set(range(bs[b], bs[b + 1])) <= set(toks.tolist())
    # the budget exactly at a block boundary of the score order
    order = sorted(range(len(sc)), key=lambda b: (-sc[b], b))
    budget = sum(bs[b + 1] - bs[b] for b in order[:5])
    assert np.array_equal(O.select_whole_blocks(sc, bs, budget)[3], O.select_tokens(sc, bs, budget))

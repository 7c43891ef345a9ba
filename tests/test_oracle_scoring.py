"""Pins for oracle O1 (Algorithm 1) and O2 (weight table, T7).

Every check compares the oracle with something other than itself: closed
forms, SPEC worked examples, a brute-force loop on tiny inputs, a library
softmax, invariants.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def random_causal_attention(seed, L, H, S):
    r = G.rng(seed, 1)
    A = np.zeros((L, H, S, S))
    for l in range(L):
        for h in range(H):
            for q in range(S):
                w = r.random(q + 1) ** 3
                A[l, h, q, : q + 1] = w / w.sum()
    return A


def test_causal_attention_is_a_valid_attention_map():
    # AttentionTensor invariants: causal, rows sum to 1, non-negative.
    Qs, Ks = G.scoring_qk(0, 2, 40, 4, 2, 16)
    A = O.causal_attention(Qs, Ks)
    assert np.all(A >= 0)
    assert np.allclose(A.sum(-1), 1.0, atol=1e-12)
    assert np.all(np.triu(A, 1) == 0)


def test_causal_attention_matches_torch_softmax():
    # Library routine: torch softmax over masked logits (float64).
    Qs, Ks = G.scoring_qk(1, 1, 33, 4, 2, 16)
    A = O.causal_attention(Qs, Ks)
    q = torch.tensor(Qs[0], dtype=torch.float64).permute(1, 0, 2)          # [H, S, d]
    k = torch.tensor(Ks[0], dtype=torch.float64).permute(1, 0, 2).repeat_interleave(2, 0)
    z = q @ k.transpose(1, 2) / math.sqrt(16)
    z = z.masked_fill(~torch.ones(33, 33, dtype=torch.bool).tril(), float("-inf"))
    ref = torch.softmax(z, dim=-1).numpy()
    assert np.allclose(A[0], ref, atol=1e-14)


def test_full_mass_in_overlap_gives_one():
    # every future query puts all its mass inside O_i -> s_i = 1.0.
    S, W, R = 40, 8, 16
    i = 20
    A = np.zeros((1, 1, S, S))
    for q in range(S):
        A[0, 0, q, max(0, q - 3): q + 1] = 1.0 / (q + 1 - max(0, q - 3))
    for q in range(i + 1, i + W + 1):
        A[0, 0, q, :] = 0
        A[0, 0, q, i - 5: i + 1] = 1.0 / 6
    s, ov, dr = O.score_positions_from_attention(A, [i], W, R, 1.0)[i]
    assert s == pytest.approx(1.0, abs=1e-15) and dr == 0.0


def test_full_mass_on_position_zero_gives_minus_alpha():
    # i >= R and all future mass on position 0 -> s_i = -alpha.
    S, W, R = 64, 8, 16
    i = 30
    A = np.zeros((2, 3, S, S))
    A[:, :, :, 0] = 1.0
    for alpha in (1.0, 0.5, 2.0):
        s, ov, dr = O.score_positions_from_attention(A, [i], W, R, alpha)[i]
        assert s == pytest.approx(-alpha, abs=1e-15)


def brute_force_scores(A, cands, W, R, alpha):
    """Quadruple loop over (l, h, q, k) straight from Alg.1 line 3-8 with the
    set memberships written as inequalities."""
    L, H, S, _ = A.shape
    out = {}
    for i in cands:
        tot_o = tot_d = 0.0
        n = 0
        for l in range(L):
            for h in range(H):
                for q in range(S):
                    if not (i + 1 <= q <= i + W):
                        continue
                    n += 1
                    for k in range(S):
                        if i - R + 1 <= k <= i:
                            tot_o += A[l, h, q, k]
                        elif k <= i - R:
                            tot_d += A[l, h, q, k]
        if n:
            out[i] = (tot_o - alpha * tot_d) / n
    return out


def test_spec_brute_force_example():
    # random causal tensor S=64, L=2, H=2, seed 42; candidates {8,31,60}; W=8, R=16.
    A = random_causal_attention(42, 2, 2, 64)
    got = O.score_positions_from_attention(A, [8, 31, 60], 8, 16, 1.0)
    ref = brute_force_scores(A, [8, 31, 60], 8, 16, 1.0)
    assert set(got) == set(ref)
    for i in ref:
        assert got[i][0] == pytest.approx(ref[i], abs=1e-9)


@pytest.mark.parametrize("seed", range(20))
def test_brute_force_random(seed):
    r = G.rng(seed, 2)
    S = int(r.integers(5, 48))
    L, H = int(r.integers(1, 3)), int(r.integers(1, 4))
    W, R = int(r.integers(1, 9)), int(r.integers(1, 20))
    alpha = float(r.random() * 2)
    A = random_causal_attention(seed + 100, L, H, S)
    cands = list(range(S))
    got = O.score_positions_from_attention(A, cands, W, R, alpha)
    ref = brute_force_scores(A, cands, W, R, alpha)
    assert set(got) == set(ref)            # S-1 is invalid (Q2)
    assert S - 1 not in got
    for i in ref:
        assert got[i][0] == pytest.approx(ref[i], abs=1e-9)


def test_uniform_attention_closed_form():
    # Qs = 0 => every logit is 0 => row q is uniform 1/(q+1).  Then
    # Ov = |O_i|/(q+1) = min(R, i+1)/(q+1), Dr = max(0, i-R+1)/(q+1).
    S, Hq, Hkv, d, W, R, alpha = 300, 4, 2, 16, 8, 128, 1.0
    Qs = np.zeros((1, S, Hq, d), np.float32)
    _, Ks = G.scoring_qk(3, 1, S, Hq, Hkv, d)
    tok = G.tokens(3, S)
    s = O.score_delimiters(tok, G.T7_IDS, Qs, Ks, W, R, alpha)
    dset = set(G.T7_IDS.tolist())
    n_checked = 0
    for i in range(S):
        if tok[i] in dset and i <= S - 2:
            F = range(i + 1, min(i + W, S - 1) + 1)
            expect = np.mean([(min(R, i + 1) - alpha * max(0, i - R + 1)) / (q + 1) for q in F])
            assert s[i] == pytest.approx(expect, abs=1e-12)
            n_checked += 1
        else:
            assert np.isnan(s[i])
    assert n_checked > 20


def test_qk_path_equals_attention_map_path():
    S, Hq, Hkv, d = 90, 4, 2, 16
    Qs, Ks = G.scoring_qk(5, 2, S, Hq, Hkv, d)
    tok = G.tokens(5, S)
    s = O.score_delimiters(tok, G.T7_IDS, Qs, Ks, 8, 20, 1.0)
    A = O.causal_attention(Qs, Ks)
    cands = [i for i in range(S) if tok[i] in set(G.T7_IDS.tolist())]
    ref = O.score_positions_from_attention(A, cands, 8, 20, 1.0)
    for i, (si, _, _) in ref.items():
        assert s[i] == pytest.approx(si, abs=1e-12)
    # sampled entry point gives identical values
    sub = cands[::3]
    s2 = O.score_delimiters(tok, G.T7_IDS, Qs, Ks, 8, 20, 1.0, candidates=sub)
    for i in sub:
        if i in ref:
            assert s2[i] == s[i]


def test_bounds_and_alpha_monotone():
    # s_i in [-alpha, 1]; non-increasing in alpha.
    A = random_causal_attention(7, 1, 2, 200)
    cands = list(range(0, 199, 7))
    prev = None
    for alpha in (0.0, 0.5, 1.0, 2.0):
        res = O.score_positions_from_attention(A, cands, 8, 32, alpha)
        for i, (s, ov, dr) in res.items():
            assert -alpha - 1e-12 <= s <= 1 + 1e-12
            assert ov + dr <= 1 + 1e-12
            if prev is not None:
                assert s <= prev[i] + 1e-15
        prev = {i: v[0] for i, v in res.items()}


def test_overlap_drop_future_partition_rows():
    # O_i, D_i and (i, q] partition [0, q]: Ov + Dr + Fut = 1 for every row
    # (this identity is what the GPU's LSE+band reformulation relies on).
    A = random_causal_attention(9, 1, 1, 300)
    for i in (0, 5, 127, 128, 200, 290):
        F, Oi, Di = O.regions(i, 300, 8, 128)
        for q in F:
            fut = A[0, 0, q, i + 1: q + 1].sum()
            tot = A[0, 0, q, Oi].sum() + (A[0, 0, q, Di].sum() if Di else 0) + fut
            assert tot == pytest.approx(1.0, abs=1e-12)
        assert sorted(Oi + Di) == list(range(i + 1))


# ---------------------------------------------------------------------------
# O2 weight table
# ---------------------------------------------------------------------------
def _seq_with_means(ids, means, reps=3):
    toks, s = [], []
    for t, m in zip(ids, means):
        for r in range(reps):
            toks.append(t)
            s.append(m + (r - 1) * 0.01)    # mean over reps is m
        toks.append(5)                       # filler
        s.append(np.nan)
    return np.array(toks), np.array(s)


def test_table_singleton_is_one():
    # one token id, one valid score -> weight 1.0.
    w10, _ = O.weight_table(np.array([28723, 3]), np.array([-0.3, np.nan]), [28723, 28725])
    assert w10.tolist() == [10, 0]


def test_table_minmax_endpoints():
    # means 0.2 and 0.8 under minmax -> 0.0 and 1.0.
    toks, s = _seq_with_means([28723, 28725], [0.2, 0.8], reps=1)
    w10, means = O.weight_table(toks, s, [28723, 28725])
    assert w10.tolist() == [0, 10]


def test_table_reproduces_paper_table7():
    # Table 7 is a fixed point of the rule: give each delimiter
    # id a mean score equal to its printed weight plus an anchor id at 0.0;
    # min-max over [0, 1] and rounding to tenths returns the printed weights.
    gold = json.load(open(os.path.join(GOLD, "t7_mistral_weights.json")))
    ids = gold["token_ids"] + [777]
    means = gold["weights"] + [0.0]
    toks, s = _seq_with_means(ids, means)
    w10, _ = O.weight_table(toks, s, ids)
    assert [w / 10 for w in w10[:-1].tolist()] == gold["weights"]
    assert G.T7_IDS.tolist() == gold["token_ids"]
    assert [w / 10 for w in G.T7_W10.tolist()] == gold["weights"]


def test_table_round_half_up_and_nan_ignored():
    # binary-exact means: 10w = 2.5 -> 3 (half-up, not half-even), 7.5 -> 8
    toks, s = _seq_with_means([1, 2, 3, 4], [0.0, 0.25, 0.75, 1.0], reps=1)
    w10, _ = O.weight_table(toks, s, [1, 2, 3, 4, 9])
    assert w10.tolist() == [0, 3, 8, 10, 0]        # id 9 absent -> 0


def test_table_invariant_to_affine_score_change():
    # min-max makes the table invariant to s -> a*s + b (a > 0).
    r = G.rng(11)
    toks = r.choice(np.array([1, 2, 3, 4, 5]), size=200)
    s = r.standard_normal(200)
    w1, _ = O.weight_table(toks, s, [1, 2, 3, 4, 5])
    w2, _ = O.weight_table(toks, 4.0 * s + 2.0, [1, 2, 3, 4, 5])
    assert w1.tolist() == w2.tolist()

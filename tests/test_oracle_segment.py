"""Pins for oracle O3 (DD-Select, Delta = 14 at P:328) and O4
(uniform page mapping)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import dynsplit_oracle as O
from synth import generators as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def spans(starts):
    return [[int(a), int(b)] for a, b in zip(starts[:-1], starts[1:])]


def build_seq(L, delims):
    toks = np.full(L, 5, np.int32)
    ids, w10 = [], []
    for k, (pos, w) in enumerate(delims):
        toks[pos] = 1000 + k
        ids.append(1000 + k)
        w10.append(w)
    return toks, ids, w10


@pytest.mark.parametrize("name", ["fallback_fixed_intervals", "three_delimiters"])
def test_golden_examples(name):
    ex = json.load(open(os.path.join(GOLD, "segment_examples.json")))[name]
    toks, ids, w10 = build_seq(ex["L"], ex["delimiters"])
    got = O.segment(toks, ids, w10, ex["C"], ex["delta"], *ex["lambda"])
    assert spans(got) == ex["expected_spans"]


def test_dominant_delimiter_at_initial_end():
    # one delimiter with w=1 exactly at s_e is chosen for any lambda.
    toks, ids, w10 = build_seq(200, [(32, 10), (25, 9), (40, 9)])
    for lam in [(0, 1), (1, 3), (1, 2), (1, 1)]:
        got = O.segment(toks, ids, w10, 32, 14, *lam)
        assert got[1] == 32


def test_delta_zero_is_fixed_intervals():
    toks = G.tokens(1, 500)
    got = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 0)
    assert got == list(range(0, 500, 32)) + [500]


def check_length_law(starts, S, C, delta):
    assert starts[0] == 0 and starts[-1] == S
    lens = np.diff(starts)
    assert np.all(lens >= 1)
    assert np.all(lens[:-1] >= C - delta) and np.all(lens[:-1] <= C + delta)
    assert lens[-1] <= C + delta


@pytest.mark.parametrize("seed", range(40))
def test_length_law_random(seed):
    # S:217 / S:519: non-final spans in [C-D, C+D], tiling [0, L).
    r = G.rng(seed, 7)
    S = int(r.integers(1, 2000))
    C = int(r.integers(2, 80))
    delta = int(r.integers(0, C))
    lam_den = int(r.integers(1, 6))
    lam_num = int(r.integers(0, lam_den + 1))
    toks = G.tokens(seed, S)
    w10 = r.integers(0, 11, size=G.T7_IDS.size)
    starts = O.segment(toks, G.T7_IDS, w10, C, delta, lam_num, lam_den)
    check_length_law(starts, S, C, delta)


def exact_key(w10, e, s_e, delta, lam):
    return lam * Fraction(int(w10), 10) + (1 - lam) * (1 - Fraction(abs(e - s_e), delta + 1))


@pytest.mark.parametrize("seed", range(30))
def test_each_cut_is_the_exhaustive_argmax(seed):
    # S:204 (brute force over the window at each step): every cut e* must be
    # a boundary token maximising the exact key in its window with no smaller
    # position attaining the same key; or s_e when the window holds none.
    r = G.rng(seed, 8)
    S = int(r.integers(50, 800))
    C = int(r.integers(8, 64))
    delta = int(r.integers(0, C))
    lam = Fraction(int(r.integers(0, 5)), 4)
    toks = G.tokens(seed + 1000, S, inner_rate=float(r.random() * 0.4))
    w10 = r.integers(0, 11, size=G.T7_IDS.size)
    wmap = dict(zip(G.T7_IDS.tolist(), w10.tolist()))
    starts = O.segment(toks, G.T7_IDS, w10, C, delta, lam.numerator, lam.denominator)
    for s_c, e_star in zip(starts[:-2], starts[1:-1]):
        s_e = s_c + C
        window = [e for e in range(s_e - delta, s_e + delta + 1)
                  if s_c + 1 <= e <= S - 1 and int(toks[e]) in wmap]
        if not window:
            assert e_star == s_e
            continue
        keys = {e: exact_key(wmap[int(toks[e])], e, s_e, delta, lam) for e in window}
        best = max(keys.values())
        assert keys.get(e_star) == best
        assert all(keys[e] < best for e in window if e < e_star)
    check_length_law(starts, S, C, delta)


def test_lambda_zero_ignores_weights():
    # lambda = 0 -> plan depends only on delimiter positions.
    toks = G.tokens(4, 3000)
    a = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14, 0, 1)
    b = O.segment(toks, G.T7_IDS, np.full(13, 3), 32, 14, 0, 1)
    assert a == b


def test_lambda_one_picks_unique_max_weight():
    # lambda = 1 and a unique max-weight delimiter in the window.
    toks, ids, w10 = build_seq(100, [(20, 4), (27, 10), (33, 6), (40, 9)])
    got = O.segment(toks, ids, w10, 32, 14, 1, 1)
    assert got[1] == 27


def test_float_key_agrees_except_on_exact_ties():
    # The literal float64 formula picks the same cut as the exact key
    # wherever the window's best exact key is unique; where the two plans
    # first diverge, both cuts must carry the same exact key (a tie that
    # float rounding ordered differently) -- the reason O3 uses rationals.
    n_div = 0
    for seed in range(10):
        toks = G.tokens(seed, 4000)
        w10 = G.rng(seed, 9).integers(0, 11, size=13)
        wmap = dict(zip(G.T7_IDS.tolist(), w10.tolist()))
        for lam in (Fraction(1, 2), Fraction(1, 3)):
            a = O.segment(toks, G.T7_IDS, w10, 32, 14, lam.numerator, lam.denominator)
            b = O.segment_float_key(toks, G.T7_IDS, w10, 32, 14, float(lam))
            if a == b:
                continue
            n_div += 1
            k = next(j for j in range(min(len(a), len(b))) if a[j] != b[j])
            s_e = a[k - 1] + 32
            ka = exact_key(wmap[int(toks[a[k]])], a[k], s_e, 14, lam)
            kb = exact_key(wmap[int(toks[b[k]])], b[k], s_e, 14, lam)
            assert ka == kb and a[k] < b[k]
    assert n_div < 20


def test_empty_sequence_and_bad_delta_raise():
    with pytest.raises(ValueError):
        O.segment(np.zeros(0, np.int32), G.T7_IDS, G.T7_W10, 32, 14)
    with pytest.raises(ValueError):
        O.segment(np.zeros(10, np.int32), G.T7_IDS, G.T7_W10, 8, 8)


def test_single_block_and_tiny_sequences():
    for S in (1, 2, 31, 32, 33):
        got = O.segment(G.tokens(S, S), G.T7_IDS, G.T7_W10, 32, 14)
        check_length_law(got, S, 32, 14)
        if S <= 32:
            assert got == [0, S]


# ---------------------------------------------------------------------------
# O4 uniform mapping (bijection, inverse, page counts)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(10))
def test_page_map_bijection(seed):
    r = G.rng(seed, 10)
    S = int(r.integers(1, 700))
    P = int(r.choice([4, 8, 16, 32]))
    starts = O.segment(G.tokens(seed, S), G.T7_IDS, G.T7_W10, 32, 14)
    pf, pb, pv = O.page_map(starts, P)
    lens = np.diff(starts)
    assert pf[-1] == sum(-(-int(l) // P) for l in lens)
    assert pv.sum() == S and np.all(pv >= 1) and np.all(pv <= P)
    slots = set()
    for b in range(len(lens)):
        for t in range(starts[b], starts[b + 1]):
            o = t - starts[b]
            pg, sl = pf[b] + o // P, o % P
            assert pb[pg] == b and sl < pv[pg]
            slots.add((pg, sl))
    assert len(slots) == S                          # every token exactly once
    X = r.standard_normal((S, 3, 5))
    Xp = O.repack(X, starts, P)
    assert np.array_equal(O.unpack(Xp, starts, P), X)
    used = np.zeros(Xp.shape[1:3], bool)
    for pg, sl in slots:
        used[pg, sl] = True
    assert np.all(Xp[:, ~used, :] == 0)           # padding slots are zero


# ---------------------------------------------------------------- NEXT-1: incremental update
def test_incremental_extend_by_zero_is_identity():
    # S:212
    toks = G.tokens(41, 300)
    prev = O.segment(toks, G.T7_IDS, G.T7_W10, 64, 14)
    new, f = O.segment_incremental(prev, toks, G.T7_IDS, G.T7_W10, 64, 14)
    assert new == prev and f == len(prev) - 1


def test_incremental_frozen_prefix_numbers():
    # S:213 with the strict frozen rule (Q23): L' = 300, C = 64, Delta = 14 ->
    # every block starting at s_c < 222 is kept verbatim
    toks = G.tokens(42, 301)
    prev = O.segment(toks[:300], G.T7_IDS, G.T7_W10, 64, 14)
    new, f = O.segment_incremental(prev, toks, G.T7_IDS, G.T7_W10, 64, 14)
    kept = [s for s in prev[:-1] if s + 64 + 14 < 300]
    assert new[:len(kept)] == kept and f == len(kept)


@pytest.mark.parametrize("seed", range(6))
def test_incremental_equals_from_scratch(seed):
    # random prefixes L' in [100, 500] extended by 1..64 tokens (plus
    # chained one-token steps): identical to segmenting the whole sequence
    r = G.rng(7, seed)
    for trial in range(40):
        C = int(r.choice([16, 32, 64]))
        delta = int(r.integers(0, C))
        Lp = int(r.integers(100, 501))
        L = Lp + int(r.integers(1, 65))
        toks = G.tokens(1000 * seed + trial, L)
        w10 = r.integers(0, 11, size=len(G.T7_IDS)).astype(np.uint8)
        prev = O.segment(toks[:Lp], G.T7_IDS, w10, C, delta)
        new, f = O.segment_incremental(prev, toks, G.T7_IDS, w10, C, delta)
        assert new == O.segment(toks, G.T7_IDS, w10, C, delta), (seed, trial, C, delta, Lp, L)
        assert new[:f] == prev[:f]
    # token-by-token decoding
    toks = G.tokens(77 + seed, 400)
    plan = O.segment(toks[:200], G.T7_IDS, G.T7_W10, 32, 14)
    for L in range(201, 401):
        plan, _ = O.segment_incremental(plan, toks[:L], G.T7_IDS, G.T7_W10, 32, 14)
    assert plan == O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)


def test_incremental_rejects_shorter_sequence():
    toks = G.tokens(43, 200)
    prev = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
    with pytest.raises(ValueError):
        O.segment_incremental(prev, toks[:150], G.T7_IDS, G.T7_W10, 32, 14)

"""Pins for oracle O10 (NEXT-3): the KV Reuse Steps 1-3 of Appendix B.2
(SPEC plan_reuse / decode_loop), the page sets of the
paged realisation, and the offloaded decode loop's accounting."""
import json
import os

import numpy as np
import pytest

from oracle import dynsplit_oracle as O
from synth import generators as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_plan_reuse_worked_example():
    ex = json.load(open(os.path.join(GOLD, "reuse_examples.json")))
    n, reused, fresh = O.plan_reuse(ex["prev"], ex["next"], truncate=True)
    assert n == ex["truncated"]["reuse_len"]
    assert [r.tolist() for r in reused] == ex["truncated"]["reused"]
    assert [f.tolist() for f in fresh] == ex["truncated"]["fresh"]
    n, reused, fresh = O.plan_reuse(ex["prev"], ex["next"], truncate=False)
    assert [r.tolist() for r in reused] == ex["untruncated"]["reused"]
    assert [f.tolist() for f in fresh] == ex["untruncated"]["fresh"]


def test_plan_reuse_spec_examples():
    """identical steps reuse everything; a head disjoint from its
    previous selection forces reuse_len = 0 everywhere."""
    sel = [np.arange(0, 64, 2), np.arange(1, 65, 2), np.arange(100, 132)]
    n, reused, fresh = O.plan_reuse(sel, sel)
    assert n == 32 and all(len(f) == 0 for f in fresh)
    assert all(np.array_equal(r, s) for r, s in zip(reused, sel))
    nxt = [sel[0], sel[1], np.arange(200, 232)]
    n, reused, fresh = O.plan_reuse(sel, nxt)
    assert n == 0 and all(np.array_equal(f, s) for f, s in zip(fresh, nxt))
    with pytest.raises(ValueError):
        O.plan_reuse(sel, sel[:2])


@pytest.mark.parametrize("truncate", [True, False])
def test_plan_reuse_random_drift(truncate):
    """over 50 drifting steps reused + fresh rebuilds next exactly,
    reused comes from the previous step, the parts are disjoint; with
    truncation every head reuses the same number of entries, the largest r
    such that every head has r common entries (counted with python sets), and
    they are its r smallest common entries."""
    rng = np.random.default_rng(9)
    H, S, k = 4, 512, 64
    prev = [np.sort(rng.choice(S, k, replace=False)) for _ in range(H)]
    for _ in range(50):
        nxt = []
        for p in prev:
            keep = rng.choice(p, k - 8, replace=False)
            new = rng.choice(np.setdiff1d(np.arange(S), keep), 8, replace=False)
            nxt.append(np.sort(np.concatenate([keep, new])))
        n, reused, fresh = O.plan_reuse(prev, nxt, truncate)
        common = [sorted(set(p.tolist()) & set(q.tolist())) for p, q in zip(prev, nxt)]
        for h in range(H):
            assert sorted(reused[h].tolist() + fresh[h].tolist()) == nxt[h].tolist()
            assert set(reused[h].tolist()) <= set(prev[h].tolist())
            assert not set(reused[h].tolist()) & set(fresh[h].tolist())
        if truncate:
            r = 0
            while all(len(c) > r for c in common):
                r += 1
            assert n == r and all(reused[h].tolist() == common[h][:r] for h in range(H))
        else:
            assert all(reused[h].tolist() == common[h] for h in range(H))
        prev = nxt


def test_pages_of_tokens_bruteforce():
    """The page of every token, found by scanning page_map's (page_block,
    page_valid) runs -- an independent walk of the page layout."""
    toks = G.tokens(11, 900)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
    for P in (8, 16, 32):
        pf, pb, pv = O.page_map(starts, P)
        owner = {}
        t = 0
        for j in range(len(pb)):          # pages are laid out in token order, each holds pv[j] tokens
            for _ in range(int(pv[j])):
                owner[t] = j
                t += 1
        assert t == 900
        rng = np.random.default_rng(P)
        sel = np.sort(rng.choice(900, 123, replace=False))
        assert O.pages_of_tokens(sel, starts, P).tolist() == sorted({owner[int(x)] for x in sel})
        assert O.group_pages([sel[:50], sel[40:]], starts, P).tolist() == sorted({owner[int(x)] for x in sel})


def test_offload_loop_accounting():
    """Identical queries move nothing after the first step (without
    truncation); drifting queries: every step reused + fresh = the KV head's
    page set, and the outputs are the plain decode step's (reuse only decides
    what is moved); a budget >= S needs every page each step."""
    S, Hq, Hkv, d = 700, 4, 2, 32
    toks = G.tokens(12, S)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
    q, K, V = G.decode_qkv(12, S, Hq, Hkv, d)
    steps = O.offload_decode_loop([q, q, q], K, V, starts, 100, truncate=False)
    assert all(len(f) == 0 for st in steps[1:] for f in st["fresh"])
    assert all(len(f) > 0 for f in steps[0]["fresh"])
    rng = np.random.default_rng(3)
    qs = [q]
    for _ in range(4):
        qs.append(0.95 * qs[-1] + 0.3 * rng.standard_normal(q.shape))
    for trunc in (True, False):
        steps = O.offload_decode_loop(qs, K, V, starts, 100, truncate=trunc)
        for i, st in enumerate(steps):
            ref = O.decode_step(qs[i], K, V, starts, 100)
            assert np.array_equal(st["o"], ref["o"]) and np.array_equal(st["lse"], ref["lse"])
            for hk in range(Hkv):
                assert sorted(st["reused"][hk].tolist() + st["fresh"][hk].tolist()) == st["pages"][hk].tolist()
    n_pages = int(O.page_map(starts, 16)[0][-1])
    steps = O.offload_decode_loop(qs[:2], K, V, starts, S, truncate=True)
    assert all(len(p) == n_pages for p in steps[1]["pages"])
    assert steps[1]["reuse_len"] == n_pages and all(len(f) == 0 for f in steps[1]["fresh"])

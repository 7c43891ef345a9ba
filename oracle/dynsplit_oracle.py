"""DynSplit-KV CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct float64 (numpy) implementation of everything the
B200 hot path computes, written from the paper (arXiv 2602.03184,
/root/reference/PAPER.md, cited as ``P:<line>``) with SPEC.md (``S:<line>``)
used only for interfaces and worked examples.  Readings of ambiguous passages
follow SURVEY.md section 8(c) (``Qn``) and are listed in DESIGN.md.

Who may import this module: ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``).  The product
path (``paper_2602_03184_b200``) never imports, links or executes it, and this
module never imports the product path.  It shares no code, tables or constants
with the CUDA sources.

Conventions (one sequence at a time; batch loops live in the callers):
  tokens  : int array [S]
  Qs      : float [Ls, S, Hq, d]   (queries of the scored layers)
  Ks      : float [Ls, S, Hkv, d]  (keys of the scored layers)
  K, V    : float [S, Hkv, d]      (one layer's KV cache, token-major)
  q       : float [Hq, d]          (decode query of one step)
  query head h reads KV head h // (Hq // Hkv)   (GQA, Q3)
All float inputs are converted to float64 exactly (bf16/fp32 values are exactly
representable); every computation below is float64 unless stated.

Pinned by tests/test_oracle_*.py.  Functions without an independent pin would
say "parity unpinned" here; at present every function below has at least one
pin ("Oracle pins").
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

__all__ = [
    "regions", "causal_attention", "score_positions_from_attention",
    "score_delimiters", "weight_table", "segment", "segment_float_key",
    "page_map", "repack", "unpack", "digests", "block_scores",
    "token_scores", "select_tokens", "selection_from_tokens",
    "select_blocks_direct", "sparse_attention", "dense_attention",
    "merge_partials", "decode_step", "plan_reuse", "pages_of_tokens", "group_pages",
    "offload_decode_loop",
]


def _f64(x):
    return np.asarray(x, dtype=np.float64)


# ---------------------------------------------------------------------------
# O1  Delimiter importance scoring, Algorithm 1, eq. at P:176-184,
#     W=8, R=128, alpha=1.
# ---------------------------------------------------------------------------
def regions(i: int, S: int, W: int, R: int):
    """Algorithm 1 lines 3-5 for candidate position i.

    F_i = {i+1 .. i+W} clipped to S-1 (Q2: an empty F_i makes i invalid).
    O_i = {max(0, i-R+1) .. i}.
    D_i = {0 .. i-R}, empty when i < R (Q1: P:158's max(0, i-R) would put
    position 0 in both O_i and D_i; O_i and D_i partition {0..i}).
    """
    F = list(range(i + 1, min(i + W, S - 1) + 1))
    O = list(range(max(0, i - R + 1), i + 1))
    D = list(range(0, i - R + 1)) if i >= R else []
    return F, O, D


def causal_attention(Qs, Ks, scale=None):
    """The attention maps A^{(l,h)} of Algorithm 1 line 1.

    A[l,h,q,k] = softmax_k( Qs[l,q,h] . Ks[l,k,h//g] * scale ) over k <= q,
    0 for k > q.  scale = 1/sqrt(d) (Q3).  Max-subtracted softmax (Q20).
    Returns float64 [Ls, Hq, S, S].  Memory O(S^2): small S only.
    """
    Qs = _f64(Qs)
    Ks = _f64(Ks)
    Ls, S, Hq, d = Qs.shape
    Hkv = Ks.shape[2]
    g = Hq // Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    A = np.zeros((Ls, Hq, S, S))
    mask = np.tril(np.ones((S, S), dtype=bool))
    for l in range(Ls):
        for h in range(Hq):
            Z = (Qs[l, :, h, :] @ Ks[l, :, h // g, :].T) * scale
            Z = np.where(mask, Z, -np.inf)
            Z = Z - Z.max(axis=1, keepdims=True)
            E = np.exp(Z)
            A[l, h] = E / E.sum(axis=1, keepdims=True)
    return A


def score_positions_from_attention(A, candidates, W=8, R=128, alpha=1.0):
    """Algorithm 1 lines 2-9 on given attention maps A [L, H, S, S].

    OverlapCBD_i = E_{l,h,q in F_i} sum_{k in O_i} A_qk
    DropCBD_i    = E_{l,h,q in F_i} sum_{k in D_i} A_qk
    s_i = OverlapCBD_i - alpha * DropCBD_i
    E is the uniform mean over all (l, h, q) triples (Q3).
    Returns {i: (s_i, overlap, drop)} for valid candidates only (Q2).
    """
    A = _f64(A)
    L, H, S, _ = A.shape
    out = {}
    for i in candidates:
        F, O, D = regions(int(i), S, W, R)
        if not F:
            continue
        ov = 0.0
        dr = 0.0
        n = 0
        for l in range(L):
            for h in range(H):
                for q in F:
                    ov += A[l, h, q, O].sum()
                    if D:
                        dr += A[l, h, q, D].sum()
                    n += 1
        ov /= n
        dr /= n
        out[int(i)] = (ov - alpha * dr, ov, dr)
    return out


def _attention_rows(Qs_lh, Ks_lh, rows, scale):
    """Softmax rows q in `rows` of one (layer, head): p[q, k] for k <= q."""
    out = {}
    for q in rows:
        z = (Ks_lh[: q + 1] @ Qs_lh[q]) * scale
        z = z - z.max()
        e = np.exp(z)
        out[q] = e / e.sum()
    return out


def score_delimiters(tokens, delim_ids, Qs, Ks, W=8, R=128, alpha=1.0,
                     candidates=None):
    """Per-position delimiter scores s_i of Algorithm 1 for one sequence.

    Candidate positions D (Alg.1 input) are the positions whose token id is in
    the semantic-boundary set B (Q27); positions with empty F_i are
    invalid (Q2).  Attention rows are computed straight from Qs/Ks (the
    attention maps the model would produce) one row at a time.
    `candidates` restricts the work to a subset (sampled full-size parity).
    Returns float64 [S] with NaN where i is not a valid candidate.
    """
    tokens = np.asarray(tokens)
    Qs = _f64(Qs)
    Ks = _f64(Ks)
    Ls, S, Hq, d = Qs.shape
    Hkv = Ks.shape[2]
    g = Hq // Hkv
    scale = 1.0 / math.sqrt(d)
    dset = {int(t) for t in delim_ids}
    if candidates is None:
        candidates = [i for i in range(S) if int(tokens[i]) in dset]
    cand = [int(i) for i in candidates if i <= S - 2 and int(tokens[i]) in dset]
    rows = sorted({q for i in cand for q in regions(i, S, W, R)[0]})
    s = np.full(S, np.nan)
    if not cand:
        return s
    acc = {i: 0.0 for i in cand}
    cnt = {i: 0 for i in cand}
    for l in range(Ls):
        for h in range(Hq):
            P = _attention_rows(Qs[l, :, h, :], Ks[l, :, h // g, :], rows, scale)
            for i in cand:
                F, O, D = regions(i, S, W, R)
                for q in F:
                    p = P[q]
                    ov = p[O].sum()
                    dr = p[D].sum() if D else 0.0
                    acc[i] += ov - alpha * dr
                    cnt[i] += 1
    for i in cand:
        s[i] = acc[i] / cnt[i]
    return s


# ---------------------------------------------------------------------------
# O2  Position scores -> per-token-id weights in tenths (T7 P:720-736;
#     aggregation rule Q5 after S:150).
# ---------------------------------------------------------------------------
def weight_table(tokens, s, delim_ids):
    """w_i in [0,1] for each boundary token id, rounded to tenths (T7).

    mean of the valid s_i at that id's positions (position order), min-max
    normalised over the ids present (a single id, or all means equal, gives
    1.0), rounded half-up to tenths: w10 = floor(10 w + 0.5).  Ids with no
    valid score get w10 = 0 (reading R-P2 in DESIGN.md).
    Returns (w10 uint8 [n_ids], means dict id_index -> mean).
    """
    tokens = np.asarray(tokens)
    s = _f64(s)
    index = {int(t): j for j, t in enumerate(delim_ids)}
    sums = [0.0] * len(delim_ids)
    cnts = [0] * len(delim_ids)
    for pos in range(len(tokens)):
        j = index.get(int(tokens[pos]))
        if j is not None and not np.isnan(s[pos]):
            sums[j] += float(s[pos])
            cnts[j] += 1
    means = {j: sums[j] / cnts[j] for j in range(len(delim_ids)) if cnts[j] > 0}
    w10 = np.zeros(len(delim_ids), dtype=np.uint8)
    if means:
        lo = min(means.values())
        hi = max(means.values())
        for j, m in means.items():
            w = 1.0 if hi == lo else (m - lo) / (hi - lo)
            w10[j] = int(math.floor(10.0 * w + 0.5))
    return w10, means


# ---------------------------------------------------------------------------
# O3  DD-Select dynamic segmentation, Delta = 14.
# ---------------------------------------------------------------------------
def _dd_select_loop(tokens, delim_ids, w10, C, delta, key_fn, s_begin=0):
    S = len(tokens)
    if S < 1:
        raise ValueError("EmptySequence")
    if not (0 <= delta < C):
        raise ValueError("need 0 <= delta < C")     # S:192, Q11
    wmap = {int(t): int(w) for t, w in zip(delim_ids, w10)}
    starts = []
    s_c = s_begin                                    # step 1: current pos
    while s_c < S:
        starts.append(s_c)
        s_e = s_c + C                                # step 1: initial end
        if s_e >= S:                                 # Q12: final short chunk
            break
        best = None
        lo = max(s_e - delta, s_c + 1)               # step 2 window, Q11 clip
        hi = min(s_e + delta, S - 1)
        for e in range(lo, hi + 1):
            t = int(tokens[e])
            if t in wmap:                            # e is a boundary token
                key = key_fn(wmap[t], abs(e - s_e))
                if best is None or key > best[0]:    # ties -> smallest e (Q10)
                    best = (key, e)
        e_star = s_e if best is None else best[1]    # no boundary: e* = s_e
        s_c = e_star                                 # step 4: chunk [s, e*)
    starts.append(S)
    return starts


def segment(tokens, delim_ids, w10, C=32, delta=14, lam_num=1, lam_den=2):
    """DD-Select, evaluated in exact rational arithmetic.

    e* = argmax_{e in [s_e-D, s_e+D]} lam*w_e + (1-lam)*p_e
    w_e = w10/10 (T7 tenths), p_e = 1 - |e - s_e|/(D+1) (Q6), lam = lam_num/lam_den
    (Q7).  Chunk [s_c, e*), s_c <- e* (paper-literal, Q9).
    Returns block_starts [n_b + 1] (last entry S).
    """
    lam = Fraction(lam_num, lam_den)

    def key(w, dist):
        p = 1 - Fraction(dist, delta + 1)
        return lam * Fraction(w, 10) + (1 - lam) * p

    return _dd_select_loop(tokens, delim_ids, w10, C, delta, key)


def segment_incremental(prev_starts, tokens, delim_ids, w10, C=32, delta=14, lam_num=1, lam_den=2):
    """Incremental update during decoding ("only the most recent
    segmentation ranges are recomputed"; SPEC S:206-209 with the strict
    frozen rule of reading Q23).

    prev_starts: the plan of the prefix of length L' = prev_starts[-1];
    tokens: the extended sequence (length L >= L').  Every block whose start
    s_c satisfies s_c + C + delta < L' is kept verbatim (its window and its
    end test only see tokens < L'); segmentation resumes from the first other
    block start.  Returns (block_starts of the extended sequence, index of the
    first recomputed block).
    """
    prev = [int(x) for x in prev_starts]
    Lp, L = prev[-1], len(tokens)
    if L < Lp:
        raise ValueError("PlanMismatch: the sequence is shorter than the plan")
    if L == Lp:
        return prev, len(prev) - 1
    nprev = len(prev) - 1
    f = 0
    while f < nprev and prev[f] + C + delta < Lp:    # frozen prefix (strict <, Q23)
        f += 1
    lam = Fraction(lam_num, lam_den)

    def key(w, dist):
        p = 1 - Fraction(dist, delta + 1)
        return lam * Fraction(w, 10) + (1 - lam) * p

    s0 = prev[f] if f < nprev else Lp
    return prev[:f] + _dd_select_loop(tokens, delim_ids, w10, C, delta, key, s_begin=s0), f


def segment_float_key(tokens, delim_ids, w10, C=32, delta=14, lam=0.5):
    """Same loop with the literal float64 key (cross-check only; near-equal
    keys may round differently, which is why `segment` uses rationals)."""
    def key(w, dist):
        return lam * (w / 10.0) + (1.0 - lam) * (1.0 - dist / (delta + 1.0))

    return _dd_select_loop(tokens, delim_ids, w10, C, delta, key)


# ---------------------------------------------------------------------------
# O4  Uniform mapping of variable-length blocks onto fixed P-token pages
#     (north star; V2F "fixed-length", Q22).
# ---------------------------------------------------------------------------
def page_map(block_starts, P=16):
    """pages_b = ceil(len_b / P); page_first = exclusive prefix sum.

    page_block[j] = block of page j; page_valid[j] = min(P, len_b - P*(j - page_first[b])).
    Returns (page_first [n_b+1], page_block [n_pages], page_valid [n_pages]).
    """
    bs = [int(x) for x in block_starts]
    nb = len(bs) - 1
    page_first = [0]
    page_block = []
    page_valid = []
    for b in range(nb):
        ln = bs[b + 1] - bs[b]
        npg = -(-ln // P)
        for jj in range(npg):
            page_block.append(b)
            page_valid.append(min(P, ln - P * jj))
        page_first.append(page_first[-1] + npg)
    return (np.array(page_first, np.int64), np.array(page_block, np.int64),
            np.array(page_valid, np.int64))


def repack(X, block_starts, P=16):
    """Token t of block b at offset o -> (page page_first[b] + o//P, slot o%P).

    X [S, H, d] -> Xp [H, n_pages, P, d]; padding slots are 0.
    """
    X = _f64(X)
    S, H, d = X.shape
    page_first, _, _ = page_map(block_starts, P)
    n_pages = int(page_first[-1])
    Xp = np.zeros((H, n_pages, P, d))
    for b in range(len(block_starts) - 1):
        for t in range(int(block_starts[b]), int(block_starts[b + 1])):
            o = t - int(block_starts[b])
            Xp[:, page_first[b] + o // P, o % P, :] = X[t]
    return Xp


def unpack(Xp, block_starts, P=16):
    """Inverse of `repack`: rebuild X [S, H, d] from pages."""
    H, n_pages, _, d = Xp.shape
    S = int(block_starts[-1])
    page_first, _, _ = page_map(block_starts, P)
    X = np.zeros((S, H, d))
    for b in range(len(block_starts) - 1):
        for t in range(int(block_starts[b]), int(block_starts[b + 1])):
            o = t - int(block_starts[b])
            X[t] = Xp[:, page_first[b] + o // P, o % P, :]
    return X


# ---------------------------------------------------------------------------
# O5  V2F compression: element-wise max and min of the block's keys (
#     keys only, Q13).
# ---------------------------------------------------------------------------
def digests(K, block_starts):
    """kmax[h, b, :] = max_{t in block b} K[t, h, :], kmin likewise.

    Returns (kmax, kmin) each float64 [Hkv, n_b, d].
    """
    K = _f64(K)
    S, H, d = K.shape
    nb = len(block_starts) - 1
    kmax = np.zeros((H, nb, d))
    kmin = np.zeros((H, nb, d))
    for b in range(nb):
        blk = K[int(block_starts[b]):int(block_starts[b + 1])]
        kmax[:, b, :] = blk.max(axis=0)
        kmin[:, b, :] = blk.min(axis=0)
    return kmax, kmin


def digests_mean(K, block_starts):
    """NEXT-2 variant: mean-pooling compression ("we further evaluate our
    approach with mean pooling-based compression"; Appendix A.2,
    P:646): kmean[h, b, :] = mean over the block's tokens of K[t, h, :].
    Returns float64 [Hkv, n_b, d]."""
    K = _f64(K)
    S, H, d = K.shape
    nb = len(block_starts) - 1
    kmean = np.zeros((H, nb, d))
    for b in range(nb):
        kmean[:, b, :] = K[int(block_starts[b]):int(block_starts[b + 1])].mean(axis=0)
    return kmean


def block_scores_mean(qh, kmean_h):
    """Query-compressed vector product with the mean vector: q . kmean."""
    return (_f64(kmean_h) * _f64(qh)).sum(axis=1)


# ---------------------------------------------------------------------------
# O6  Block score = "query-compressed vector product", Q14:
#     s_b = sum_j max(q_j kmax_j, q_j kmin_j).
# ---------------------------------------------------------------------------
def block_scores(qh, kmax_h, kmin_h):
    """qh [d], kmax_h/kmin_h [n_b, d] -> float64 [n_b]."""
    qh = _f64(qh)
    return np.maximum(_f64(kmax_h) * qh, _f64(kmin_h) * qh).sum(axis=1)


# ---------------------------------------------------------------------------
# O7  Top-k selection through block-to-token mapping (Step 1
#     P:749): every token inherits its block's score, then the top `budget`
#     tokens (ties: higher score, then lower token index, Q15-Q17).
# ---------------------------------------------------------------------------
def token_scores(scores, block_starts):
    """Materialise the mapped per-token score (assign s_i to t in B_i)."""
    bs = [int(x) for x in block_starts]
    out = np.empty(bs[-1])
    for b in range(len(bs) - 1):
        out[bs[b]:bs[b + 1]] = scores[b]
    return out


def select_tokens(scores, block_starts, budget):
    """Top-`budget` tokens by (mapped score desc, token index asc), stable sort.

    Returns the selected token indices in ascending order.
    """
    ts = token_scores(_f64(scores), block_starts)
    order = np.lexsort((np.arange(len(ts)), -ts))   # primary: -score, then index
    take = order[: min(int(budget), len(ts))]
    return np.sort(take)


def selection_from_tokens(sel_tokens, scores, block_starts, budget):
    """Convert a token selection to (sel_blocks asc, marginal_block, keep).

    marginal = the block holding the last token taken in score order (the
    block that reaches the budget), keep = how many of its tokens are taken;
    (-1, 0) when every token fits in the budget.
    """
    bs = np.asarray(block_starts, np.int64)
    S = int(bs[-1])
    blk_of = np.searchsorted(bs, np.asarray(sel_tokens), side="right") - 1
    sel_blocks = sorted({int(b) for b in blk_of})
    if int(budget) >= S:
        return sel_blocks, -1, 0
    ts = token_scores(_f64(scores), block_starts)
    order = np.lexsort((np.arange(S), -ts))
    last = int(order[int(budget) - 1])
    m = int(np.searchsorted(bs, last, side="right") - 1)
    keep = int(np.sum(blk_of == m))
    return sel_blocks, m, keep


def select_blocks_direct(scores, block_starts, budget):
    """Independent block-order fill (pin for select_tokens): visit blocks by
    (score desc, index asc), take whole blocks while the budget lasts; the
    block that reaches it keeps its first tokens (Q16)."""
    bs = [int(x) for x in block_starts]
    nb = len(bs) - 1
    if bs[-1] - bs[0] <= int(budget):               # everything fits
        return (list(range(nb)), -1, 0,
                np.arange(bs[0], bs[-1], dtype=np.int64))
    order = sorted(range(nb), key=lambda b: (-float(scores[b]), b))
    remaining = int(budget)
    chosen = []
    marginal, keep = -1, 0
    for b in order:
        ln = bs[b + 1] - bs[b]
        chosen.append(b)
        if ln >= remaining:                          # this block reaches the budget
            marginal, keep = b, remaining
            break
        remaining -= ln
    toks = []
    for b in chosen:
        n = keep if b == marginal else bs[b + 1] - bs[b]
        toks.extend(range(bs[b], bs[b] + n))
    return sorted(chosen), marginal, keep, np.array(sorted(toks), np.int64)


def group_block_scores(q_group, kmax_h, kmin_h):
    """NEXT-2 group-shared GQA selection (DESIGN R23): one score per block for
    the g query heads of a KV head, the sum of the heads' V2F scores,
    sum_{h in group} sum_j max(q_hj kmax_j, q_hj kmin_j), so the group takes
    ONE selection (the paper runs GQA models; its shapes are per query
    head).  q_group [g, d]."""
    return np.sum([block_scores(qh, kmax_h, kmin_h) for qh in _f64(q_group)], axis=0)


def select_whole_blocks(scores, block_starts, budget):
    """NEXT-2 whole-block budget (DESIGN R24; "select the top-k highest-scoring
    blocks"): blocks in (score desc, index asc) order are taken whole
    until their lengths reach the budget -- the block that reaches it is taken
    whole as well (k = the fewest top blocks covering the budget).  Returns
    (ascending blocks, marginal block, its length, ascending tokens); (all,
    -1, 0, all) when every token fits."""
    bs = [int(x) for x in block_starts]
    nb = len(bs) - 1
    if bs[-1] - bs[0] <= int(budget):
        return list(range(nb)), -1, 0, np.arange(bs[0], bs[-1], dtype=np.int64)
    order = sorted(range(nb), key=lambda b: (-float(scores[b]), b))
    total = 0
    chosen = []
    for b in order:
        chosen.append(b)
        total += bs[b + 1] - bs[b]
        if total >= int(budget):
            break
    m = chosen[-1]
    toks = np.concatenate([np.arange(bs[b], bs[b + 1]) for b in sorted(chosen)]).astype(np.int64)
    return sorted(chosen), m, bs[m + 1] - bs[m], toks


# ---------------------------------------------------------------------------
# O8  Attention over the selected set (Step 3, Q20):
#     z = q.k * scale, p = softmax(z), o = sum p v, lse = log sum exp z.
# ---------------------------------------------------------------------------
def sparse_attention(qh, Kh, Vh, token_idx, scale):
    """qh [d]; Kh, Vh [S, d]; token_idx: selected tokens. Returns (o [d], lse)."""
    idx = np.asarray(token_idx, np.int64)
    if idx.size == 0:
        raise ValueError("EmptySelection")
    z = (_f64(Kh)[idx] @ _f64(qh)) * scale
    m = z.max()
    e = np.exp(z - m)
    ssum = e.sum()
    o = (e[:, None] * _f64(Vh)[idx]).sum(axis=0) / ssum
    return o, m + math.log(ssum)


def dense_attention(qh, Kh, Vh, scale):
    """Full-KV attention (the FlashAttention baseline of P:452)."""
    return sparse_attention(qh, Kh, Vh, np.arange(np.asarray(Kh).shape[0]), scale)


# ---------------------------------------------------------------------------
# O9  Log-sum-exp merge of split partials (north star: "split-K, with a
#     log-sum-exp merge"): L = log sum_s e^{lse_s}, o = sum_s e^{lse_s - L} o_s.
# ---------------------------------------------------------------------------
def merge_partials(o_parts, lse_parts):
    """o_parts [n, d], lse_parts [n] (-inf allowed for empty parts)."""
    o_parts = _f64(o_parts)
    lse_parts = _f64(lse_parts)
    m = lse_parts.max()
    if m == -np.inf:
        return np.zeros(o_parts.shape[1]), -np.inf
    w = np.exp(lse_parts - m)
    L = m + math.log(w.sum())
    o = (np.exp(lse_parts - L)[:, None] * o_parts).sum(axis=0)
    return o, L


# ---------------------------------------------------------------------------
# One decode step for one sequence and one layer (Steps 1-3).
# ---------------------------------------------------------------------------
def decode_step(q, K, V, block_starts, budget, scale=None, digest_mode="minmax", gqa_mode="head",
                budget_mode="token"):
    """q [Hq, d]; K, V [S, Hkv, d].  Per query head (Q18): O5 digests, O6
    scores, O7 selection, O8 attention.  digest_mode "mean" uses the
    mean-pooling variant.  NEXT-2 variants: gqa_mode "group"
    scores every block once per KV head with group_block_scores and the g
    query heads share that selection (R23); budget_mode "whole" takes the
    budget-reaching block whole (select_whole_blocks, R24).  Returns a dict of
    per-head results ("scores" are the scores the selection used)."""
    q = _f64(q)
    Hq, d = q.shape
    Hkv = np.asarray(K).shape[1]
    g = Hq // Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if digest_mode == "mean":
        kmean = digests_mean(K, block_starts)
    else:
        kmax, kmin = digests(K, block_starts)
    res = {"scores": [], "tokens": [], "sel_blocks": [], "marginal": [],
           "keep": [], "o": np.zeros((Hq, d)), "lse": np.zeros(Hq)}
    Kf = _f64(K)
    Vf = _f64(V)
    for h in range(Hq):
        hk = h // g
        if gqa_mode == "group":
            sc = group_block_scores(q[hk * g:(hk + 1) * g], kmax[hk], kmin[hk])
        elif digest_mode == "mean":
            sc = block_scores_mean(q[h], kmean[hk])
        else:
            sc = block_scores(q[h], kmax[hk], kmin[hk])
        if budget_mode == "whole":
            sb, m, keep, toks = select_whole_blocks(sc, block_starts, budget)
        else:
            toks = select_tokens(sc, block_starts, budget)
            sb, m, keep = selection_from_tokens(toks, sc, block_starts, budget)
        o, lse = sparse_attention(q[h], Kf[:, hk, :], Vf[:, hk, :], toks, scale)
        res["scores"].append(sc)
        res["tokens"].append(toks)
        res["sel_blocks"].append(sb)
        res["marginal"].append(m)
        res["keep"].append(keep)
        res["o"][h] = o
        res["lse"][h] = lse
    return res


# ---------------------------------------------------------------------------
# O10 Cross-step KV reuse (Appendix B.2 "KVCache Reuse with V2F", Steps 1-3,
#     P:756-765; SPEC plan_reuse / decode_loop S:379-397) and its paged,
#     host-offloaded realisation (NEXT-3; the CPU-GPU deployment, P:465-473,
#     P:583-592).
# ---------------------------------------------------------------------------
def plan_reuse(prev, nxt, truncate=True):
    """Steps 1-3 over per-head index lists prev[h] (the previous step's
    selection) and nxt[h] (this step's): per head, reusable = the ascending
    intersection of prev and next (Step 1, "compute the reusable KV for each
    head"); with truncate, reuse_len = the minimum over heads of |reusable|
    ("truncate the reusable KV based on the minimum reusable data volume ...
    a consistent length of reusable KV caches among all heads") and each
    head reuses the first reuse_len of its reusable entries in ascending index
    order (Q24 reading); without it every reusable entry is reused
    (the paged cache needs no equal lengths, DESIGN R26).  fresh = next minus
    reused (Step 2, "the truncated excess data ... combined with the new
    required data"), so reused + fresh = next per head (Step 3).  Returns
    (reuse_len, reused[h], fresh[h]); reuse_len is None without truncate."""
    if len(prev) != len(nxt):
        raise ValueError("ShapeMismatch")
    reusable = [np.intersect1d(np.asarray(p_, np.int64), np.asarray(n_, np.int64))
                for p_, n_ in zip(prev, nxt)]
    if truncate:
        reuse_len = min((len(r) for r in reusable), default=0)
        reused = [r[:reuse_len] for r in reusable]
    else:
        reuse_len = None
        reused = reusable
    fresh = [np.setdiff1d(np.asarray(n_, np.int64), u) for n_, u in zip(nxt, reused)]
    return reuse_len, reused, fresh


def pages_of_tokens(tokens, block_starts, P=16):
    """The pages (O4 ids) holding the given tokens: token t of block b at
    offset o lives in page page_first[b] + o // P (the repack rule).
    Ascending, without repeats."""
    t = np.asarray(tokens, np.int64)
    if t.size == 0:
        return np.zeros(0, np.int64)
    bs = np.asarray(block_starts, np.int64)
    pf, _, _ = page_map(block_starts, P)
    blk = np.searchsorted(bs, t, side="right") - 1
    return np.unique(pf[blk] + (t - bs[blk]) // P)


def group_pages(sel_tokens_heads, block_starts, P=16):
    """The pages a KV head must hold for its query heads' selections: the
    union of pages_of_tokens over the group (a page is stored and moved once
    per KV head, Q18)."""
    parts = [pages_of_tokens(t, block_starts, P) for t in sel_tokens_heads]
    return np.unique(np.concatenate(parts)) if parts else np.zeros(0, np.int64)


def offload_decode_loop(qs, K, V, block_starts, budget, P=16, truncate=True, reuse=True, scale=None):
    """Decode steps over one layer's fixed cache whose KV lives off the GPU
    (NEXT-3): each step is decode_step (selection and attention unchanged:
    reuse only decides what is moved, "outputs are bit-identical"); the
    KV heads' page sets (group_pages of their query heads' tokens) are planned
    against the previous step's with plan_reuse (the cache holds exactly the
    previous step's pages); reuse=False moves every needed page.  Per step:
    o, lse, pages[hk], reused[hk], fresh[hk], reuse_len."""
    Hkv = np.asarray(K).shape[1]
    out = []
    prev = None
    for q in qs:
        r = decode_step(q, K, V, block_starts, budget, scale)
        g = len(r["tokens"]) // Hkv
        pages = [group_pages(r["tokens"][hk * g:(hk + 1) * g], block_starts, P) for hk in range(Hkv)]
        if prev is None or not reuse:
            reuse_len, reused, fresh = 0, [np.zeros(0, np.int64) for _ in pages], pages
        else:
            reuse_len, reused, fresh = plan_reuse(prev, pages, truncate)
        out.append({"o": r["o"], "lse": r["lse"], "pages": pages, "reused": reused, "fresh": fresh,
                    "reuse_len": reuse_len, "tokens": r["tokens"]})
        prev = pages
    return out

"""Test infrastructure shared by the GPU parity tests: batch wrappers around
the oracle, margin certificates (SURVEY 8(c) "regime B") and comparison
helpers.  Uses only oracle/ and synth/ -- never the CUDA path's outputs as
expected values."""
from __future__ import annotations

import math

import numpy as np

from oracle import dynsplit_oracle as O
from synth import generators as G

U32 = 2.0 ** -24


def gamma(n: int) -> float:
    return n * U32 / (1 - n * U32)


def score_error_bound(qh, kmax_h, kmin_h, exact_products: bool) -> np.ndarray:
    """|fp32 block score - exact| <= gamma_n * sum_j |q_j| max(|kmax_j|, |kmin_j|)
    for ANY summation order (products of bf16 values are exact in fp32;
    fp32 inputs add one rounding per product).

    bf16 (exact products) is summed on the tensor cores as the 2d-term dot
    [q+ | q-] . [kmax | kmin] (DESIGN R22): their fp32 accumulation is not
    specified as round-to-nearest, so the bound takes n = 2d additions with
    unit roundoff 2^-23 (one truncation per addition); it also covers the
    CUDA-core kernel's d-term round-to-nearest sum."""
    d = qh.shape[-1]
    mag = (np.abs(qh.astype(np.float64)) *
           np.maximum(np.abs(kmax_h.astype(np.float64)), np.abs(kmin_h.astype(np.float64)))).sum(-1)
    if exact_products:
        n, u = 2 * d, 2.0 ** -23
        return n * u / (1 - n * u) * mag
    return gamma(d + 1) * mag


def marginal_rank(scores, starts, budget):
    lens = np.diff(np.asarray(starts))
    order = sorted(range(len(lens)), key=lambda b: (-float(scores[b]), b))
    cum = 0
    for r, b in enumerate(order):
        cum += int(lens[b])
        if cum >= budget:
            return order, r
    return order, None


def selection_certified(qh, kmax_h, kmin_h, starts, budget, exact_products=True) -> bool:
    """True if fp32 rounding of the block scores cannot change the selection
    (gap to both neighbours of the marginal block exceeds the sum of bounds)."""
    sc = O.block_scores(qh, kmax_h, kmin_h)
    if int(starts[-1] - starts[0]) <= budget:
        return True
    eps = score_error_bound(qh, kmax_h, kmin_h, exact_products)
    order, r = marginal_rank(sc, starts, budget)
    m = order[r]
    if r > 0:
        a = order[r - 1]
        if not sc[a] - sc[m] > eps[a] + eps[m]:
            return False
    if r + 1 < len(order):
        c = order[r + 1]
        if not sc[m] - sc[c] > eps[m] + eps[c]:
            return False
    return True


def certify_queries(seed, q, K, starts_list, budget, dtype="bf16", max_retry=40):
    """Resample (with derived sub-seeds) every head whose selection is not
    margin-certified.  q [B,Hq,d], K [B,S,Hkv,d] float32 arrays. Returns q."""
    q = q.copy()
    B, Hq, d = q.shape
    Hkv = K.shape[2]
    g = Hq // Hkv
    for b in range(B):
        kmax, kmin = O.digests(K[b], starts_list[b])
        for h in range(Hq):
            r = 0
            while not selection_certified(q[b, h], kmax[h // g], kmin[h // g], starts_list[b], budget,
                                          exact_products=(dtype == "bf16")):
                r += 1
                if r > max_retry:
                    raise RuntimeError("could not certify a query")
                q[b, h] = G.query_resample(seed, b, h, r, d, dtype)
    return q


def oracle_decode(q, K, V, starts_list, budget):
    """Oracle decode step for a batch: list of per-sequence result dicts."""
    return [O.decode_step(q[b], K[b], V[b], starts_list[b], budget) for b in range(q.shape[0])]


def row_rel_err(o, o_ref):
    """Per-row infinity-norm relative error (DESIGN.md tolerance Q25)."""
    o = np.asarray(o, np.float64)
    o_ref = np.asarray(o_ref, np.float64)
    num = np.abs(o - o_ref).max(axis=-1)
    den = np.maximum(np.abs(o_ref).max(axis=-1), 1e-30)
    return num / den


def starts_from_gpu(bs_row, nb):
    return [int(x) for x in bs_row[: int(nb) + 1]]


# ---------------------------------------------------------------- NEXT-2 mean-pooling mode
def mean_digest_error_bound(K, starts):
    """|fp32 mean (token-order fp32 sum, then / len) - exact mean| <=
    (gamma_len + u) * sum_t |k_t| / len, per (head, block, dim)."""
    Kf = np.abs(np.asarray(K, np.float64))
    H = Kf.shape[1]
    nb = len(starts) - 1
    out = np.zeros((H, nb, Kf.shape[2]))
    for b in range(nb):
        ln = starts[b + 1] - starts[b]
        out[:, b, :] = (gamma(ln) + U32) * Kf[starts[b]:starts[b + 1]].sum(axis=0) / ln
    return out


def score_error_bound_mean(qh, kmean_h, mean_err_h):
    """fp32 q . mean_hat: gamma_d sum_j |q_j mean_j| (one rounding per FMA) plus
    sum_j |q_j| |mean_hat_j - mean_j|, inflated 1 % for the second-order terms."""
    d = qh.shape[-1]
    qa = np.abs(np.asarray(qh, np.float64))
    return 1.01 * (gamma(d) * (qa * (np.abs(kmean_h) + mean_err_h)).sum(-1) + (qa * mean_err_h).sum(-1))


def certify_queries_mean(seed, q, K, starts_list, budget, dtype="bf16", max_retry=40):
    """certify_queries for digest_mode = mean (selection margins vs the bound above)."""
    q = q.copy()
    B, Hq, d = q.shape
    Hkv = K.shape[2]
    g = Hq // Hkv
    for b in range(B):
        st = starts_list[b]
        km = O.digests_mean(K[b], st)
        me = mean_digest_error_bound(K[b], st)
        for h in range(Hq):
            r = 0
            while True:
                sc = O.block_scores_mean(q[b, h], km[h // g])
                if int(st[-1] - st[0]) <= budget:
                    break
                eps = score_error_bound_mean(q[b, h], km[h // g], me[h // g])
                order, rk = marginal_rank(sc, st, budget)
                m = order[rk]
                ok = (rk == 0 or sc[order[rk - 1]] - sc[m] > eps[order[rk - 1]] + eps[m]) and \
                     (rk + 1 >= len(order) or sc[m] - sc[order[rk + 1]] > eps[m] + eps[order[rk + 1]])
                if ok:
                    break
                r += 1
                if r > max_retry:
                    raise RuntimeError("could not certify a query")
                q[b, h] = G.query_resample(seed, b, h, r, d, dtype)
    return q


def certify_queries_group(seed, q, K, starts_list, budget, max_retry=40):
    """Group-shared selection (DESIGN R23): the score the GPU selects on is the
    fp32 sum of the g heads' fp32 block scores.  Its error is at most the sum
    of the heads' bounds plus the g - 1 additions' rounding (2^-24 relative
    each, at most (g-1) 2^-23 sum_h |s_h|); resample the whole group (derived
    sub-seeds) until the gaps around the group's marginal block exceed the
    bounds.  q [B,Hq,d], K [B,S,Hkv,d] float32 arrays.  Returns q."""
    q = q.copy()
    B, Hq, d = q.shape
    Hkv = K.shape[2]
    g = Hq // Hkv
    for b in range(B):
        kmax, kmin = O.digests(K[b], starts_list[b])
        st = starts_list[b]
        for hk in range(Hkv):
            r = 0
            while True:
                heads = range(hk * g, (hk + 1) * g)
                s_h = [O.block_scores(q[b, h], kmax[hk], kmin[hk]) for h in heads]
                sc = np.sum(s_h, axis=0)
                eps = np.sum([score_error_bound(q[b, h], kmax[hk], kmin[hk], True) for h in heads], axis=0)
                eps = eps + (g - 1) * 2.0 ** -23 * np.sum(np.abs(s_h), axis=0)
                ok = True
                if int(st[-1] - st[0]) > budget:
                    order, rk = marginal_rank(sc, st, budget)
                    m = order[rk]
                    if rk > 0 and not sc[order[rk - 1]] - sc[m] > eps[order[rk - 1]] + eps[m]:
                        ok = False
                    if rk + 1 < len(order) and not sc[m] - sc[order[rk + 1]] > eps[m] + eps[order[rk + 1]]:
                        ok = False
                if ok:
                    break
                r += 1
                if r > max_retry:
                    raise RuntimeError("could not certify a query group")
                for h in heads:
                    q[b, h] = G.query_resample(seed + 7919, b, h, r, d, "bf16")
    return q

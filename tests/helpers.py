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
    fp32 inputs add one rounding per product)."""
    d = qh.shape[-1]
    mag = (np.abs(qh.astype(np.float64)) *
           np.maximum(np.abs(kmax_h.astype(np.float64)), np.abs(kmin_h.astype(np.float64)))).sum(-1)
    return gamma(d + (0 if exact_products else 1)) * mag


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

"""Seeded synthetic workloads for DynSplit-KV (shared by tests, bench and smoke).

This module holds NONE of the method's arithmetic: only random draws (numpy
PCG64 with recorded seeds; torch Philox on the device for bench-size caches),
rounding of values to bf16 (the storage format) and the construction of token
streams.  Both the oracle and the CUDA path consume its outputs; neither is
imported here.

Recipes:
  tokens   sentences of 1+Poisson(14) tokens ended by '.', '?' or '!'; each
           inner token is a delimiter with prob 1/7 (',' 50 %, ';' ':' 10 %,
           brackets/quotes 5 % each); other ids uniform on [0, vocab) minus
           the delimiter ids.  Delimiter ids are those of the paper's Table 7
           (Mistral-7B tokenizer).
  decode   K ~ 1.5 N(0, I), V ~ N(0, I); q_h = sqrt(rho) z_group + sqrt(1-rho) z_h;
           per (seq, KV head) `n_needles` planted tokens with
           K = c * qhat_group + 0.1 N(0, I) (S:444 idea), stored as bf16 (RNE).
  integer  ("regime A") q in {-3..3}, K in {-4..4}: every block score is an
           exact integer in fp32, ties are frequent (tests the tie rule).
  scoring  Qs, Ks ~ N(0, I) plus a slowly drifting per-position component so
           attention has local structure; bf16.
  walk     (NEXT-3) consecutive decode steps' queries as an AR(1) walk
           q_t = tau q_{t-1} + sqrt(1 - tau^2) z_t, so neighbouring steps
           select overlapping KV (the premise of cross-step reuse).
"""
from __future__ import annotations

import numpy as np

# Table 7: delimiter token ids and printed weights (tenths).
T7_IDS = np.array([28723, 609, 28804, 1101, 28745, 28747, 28725, 28742, 28808,
                   28732, 557, 28792, 28793], dtype=np.int32)
T7_W10 = np.array([10, 10, 9, 10, 7, 7, 6, 5, 9, 5, 6, 5, 5], dtype=np.uint8)

_TERMINALS = np.array([28723, 28804, 609], dtype=np.int32)      # . ? !
_TERMINAL_P = np.array([0.8, 0.1, 0.1])
_INNER = np.array([28725, 28745, 28747, 28732, 557, 28808, 28742, 28792, 28793],
                  dtype=np.int32)                                 # , ; : ( ) " ' [ ]
_INNER_P = np.array([0.5, 0.1, 0.1, 0.05, 0.05, 0.05, 0.05, 0.05, 0.05])


def rng(seed: int, *stream: int) -> np.random.Generator:
    """Named, fixed generator: numpy PCG64 seeded by SeedSequence([seed, *stream])."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), *map(int, stream)])))


def to_bf16(x) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32
    arrays holding exactly-representable bf16 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def tokens(seed: int, S: int, vocab: int = 32000, inner_rate: float = 1.0 / 7.0,
           mean_sentence: float = 14.0, delim_ids=T7_IDS) -> np.ndarray:
    """Synthetic token stream of length S (int32)."""
    r = rng(seed, 101)
    out = np.empty(S, np.int32)
    dset = set(int(t) for t in delim_ids)
    filler = np.setdiff1d(np.arange(vocab, dtype=np.int32), np.array(sorted(dset), np.int32))
    pos = 0
    while pos < S:
        n = 1 + int(r.poisson(mean_sentence))
        body = filler[r.integers(0, filler.size, size=n)]
        inner = r.random(n) < inner_rate
        body[inner] = _INNER[r.choice(_INNER.size, size=int(inner.sum()), p=_INNER_P)]
        body[-1] = _TERMINALS[r.choice(_TERMINALS.size, p=_TERMINAL_P)]
        take = min(n, S - pos)
        out[pos:pos + take] = body[:take]
        pos += take
    return out


def decode_qkv(seed: int, S: int, Hq: int, Hkv: int, d: int = 128, rho: float = 0.0,
               n_needles: int = 8, c: float = 10.0, k_scale: float = 1.5,
               dtype: str = "bf16"):
    """One sequence, one layer: q [Hq, d], K, V [S, Hkv, d] (float32 arrays
    holding bf16 values when dtype == 'bf16')."""
    r = rng(seed, 202)
    g = Hq // Hkv
    zg = r.standard_normal((Hkv, d))
    zh = r.standard_normal((Hq, d))
    q = np.sqrt(rho) * zg[np.arange(Hq) // g] + np.sqrt(1.0 - rho) * zh
    K = k_scale * r.standard_normal((S, Hkv, d))
    V = r.standard_normal((S, Hkv, d))
    for hk in range(Hkv):
        qhat = q[hk * g:(hk + 1) * g].mean(axis=0)
        qhat = qhat / max(np.linalg.norm(qhat), 1e-12)
        pos = r.choice(S, size=min(n_needles, S), replace=False)
        K[pos, hk, :] = c * qhat + 0.1 * r.standard_normal((pos.size, d))
    q, K, V = (x.astype(np.float32) for x in (q, K, V))
    if dtype == "bf16":
        q, K, V = to_bf16(q), to_bf16(K), to_bf16(V)
    return q, K, V


def decode_qkv_integer(seed: int, S: int, Hq: int, Hkv: int, d: int = 128,
                       qmax: int = 3, kmax: int = 4):
    """Regime A: integer-valued q and K (exact in bf16 and fp32), V bf16 normal."""
    r = rng(seed, 303)
    q = r.integers(-qmax, qmax + 1, size=(Hq, d)).astype(np.float32)
    K = r.integers(-kmax, kmax + 1, size=(S, Hkv, d)).astype(np.float32)
    V = to_bf16(r.standard_normal((S, Hkv, d)).astype(np.float32))
    return q, K, V


def decode_query_walk(seed: int, T: int, q0: np.ndarray, tau: float = 0.9,
                      dtype: str = "bf16") -> np.ndarray:
    """T consecutive decode-step queries [T, Hq, d] starting at q0 [Hq, d]:
    q_t = tau q_{t-1} + sqrt(1 - tau^2) z_t (z_t ~ N(0, I)), rounded to bf16."""
    r = rng(seed, 606)
    out = np.empty((T,) + q0.shape, np.float32)
    q = np.asarray(q0, np.float64)
    for t in range(T):
        if t:
            q = tau * q + np.sqrt(1.0 - tau * tau) * r.standard_normal(q.shape)
        out[t] = q
    return to_bf16(out) if dtype == "bf16" else out


def query_resample(seed: int, b: int, h: int, retry: int, d: int = 128,
                   dtype: str = "bf16") -> np.ndarray:
    """Replacement query for head h of sequence b (margin-certificate retry)."""
    r = rng(seed, 404, b, h, retry)
    q = r.standard_normal(d).astype(np.float32)
    return to_bf16(q) if dtype == "bf16" else q


def scoring_qk(seed: int, Ls: int, S: int, Hq: int, Hkv: int, d: int = 128,
               drift: float = 0.7, dtype: str = "bf16"):
    """Prefill scoring inputs Qs [Ls, S, Hq, d], Ks [Ls, S, Hkv, d]."""
    r = rng(seed, 505)
    walk = np.cumsum(r.standard_normal((Ls, S, 1, d)) * 0.05, axis=1)
    Qs = r.standard_normal((Ls, S, Hq, d)) + drift * walk
    Ks = r.standard_normal((Ls, S, Hkv, d)) + drift * walk
    Qs, Ks = Qs.astype(np.float32), Ks.astype(np.float32)
    if dtype == "bf16":
        Qs, Ks = to_bf16(Qs), to_bf16(Ks)
    return Qs, Ks


# ---------------------------------------------------------------------------
# Device-side generation for bench-size caches (torch Philox, seeded).
# ---------------------------------------------------------------------------
def torch_decode_layer(gen, S: int, Hq: int, Hkv: int, d: int, B: int, device,
                       rho: float = 0.0, n_needles: int = 8, c: float = 10.0,
                       k_scale: float = 1.5):
    """Returns q [B, Hq, d], K, V [B, S, Hkv, d] as bf16 device tensors."""
    import torch
    g = Hq // Hkv
    zg = torch.randn(B, Hkv, d, generator=gen, device=device)
    zh = torch.randn(B, Hq, d, generator=gen, device=device)
    q = (rho ** 0.5) * zg.repeat_interleave(g, dim=1) + ((1 - rho) ** 0.5) * zh
    K = torch.randn(B, S, Hkv, d, generator=gen, device=device, dtype=torch.float32)
    K.mul_(k_scale)
    qhat = q.view(B, Hkv, g, d).mean(dim=2)
    qhat = qhat / qhat.norm(dim=-1, keepdim=True).clamp_min(1e-12)
    if n_needles > 0:
        pos = torch.randint(0, S, (B, Hkv, n_needles), generator=gen, device=device)
        noise = 0.1 * torch.randn(B, Hkv, n_needles, d, generator=gen, device=device)
        vals = c * qhat[:, :, None, :] + noise
        bi = torch.arange(B, device=device)[:, None, None].expand_as(pos)
        hi = torch.arange(Hkv, device=device)[None, :, None].expand_as(pos)
        K[bi, pos, hi] = vals
    Kb = K.to(torch.bfloat16)
    del K
    V = torch.randn(B, S, Hkv, d, generator=gen, device=device, dtype=torch.float32).to(torch.bfloat16)
    return q.to(torch.bfloat16), Kb, V


def torch_query_walk(gen, T: int, q0, tau: float = 0.9):
    """Device form of decode_query_walk: [T, *q0.shape] bf16 from q0 (bf16)."""
    import torch
    out = [q0]
    q = q0.float()
    for _ in range(T - 1):
        q = tau * q + (1.0 - tau * tau) ** 0.5 * torch.randn(q.shape, generator=gen, device=q.device)
        out.append(q.to(torch.bfloat16))
    return torch.stack(out)

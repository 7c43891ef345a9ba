"""GPU parity: every row of the hot path through the C ABI vs the fp64 oracle.

Integer / index outputs (block boundaries, page maps, digests, selections)
must match bit-exactly; floating outputs within the tolerances of DESIGN.md:
attention o per-row inf-norm relative error <= 2e-3 (north star), lse within
1e-4 (absolute, scaled by max(1,|lse|)), delimiter scores within 2e-4.
"""
import math

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
    dynsplit.lib()
    return dynsplit


def t(x, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(x)).to(DEV, dtype=dtype)


def kv_dtype(name):
    return torch.bfloat16 if name == "bf16" else torch.float32


# ---------------------------------------------------------------- a3 segment
@pytest.mark.parametrize("S,C,delta,lam", [(1, 32, 14, (1, 2)), (31, 32, 14, (1, 2)),
                                           (33, 32, 14, (1, 2)), (4096, 32, 14, (1, 2)),
                                           (5003, 16, 5, (1, 3)), (20000, 64, 14, (2, 3)),
                                           (3000, 32, 0, (1, 2)), (3000, 32, 31, (0, 1)),
                                           (3000, 32, 14, (1, 1))])
def test_segment_parity(D, S, C, delta, lam):
    B = 3
    cfg = D.default_config(C=C, delta=delta, lambda_num=lam[0], lambda_den=lam[1])
    toks = np.stack([G.tokens(100 + b, S, inner_rate=0.1 + 0.1 * b) for b in range(B)])
    w10 = np.stack([G.T7_W10, G.rng(S, 5).integers(0, 11, 13), np.full(13, 5)])[:B]
    bs, nb = D.segment(t(toks), t(G.T7_IDS), t(w10.astype(np.uint8)), cfg)
    bs, nb = bs.cpu().numpy(), nb.cpu().numpy()
    mb = D.max_blocks(S, cfg)
    for b in range(B):
        ref = O.segment(toks[b], G.T7_IDS, w10[b], C, delta, *lam)
        assert nb[b] == len(ref) - 1
        assert bs[b, : nb[b] + 1].tolist() == ref
        assert np.all(bs[b, nb[b] + 1: mb + 1] == S)


# ---------------------------------------------------------------- a2 weight table
def _table_certified(toks, s, ids, margin=1e-6):
    w10, means = O.weight_table(toks, s, ids)
    if not means:
        return True
    lo, hi = min(means.values()), max(means.values())
    for m in means.values():
        if hi == lo or m in (lo, hi):
            continue
        x = 10 * (m - lo) / (hi - lo) + 0.5
        if abs(x - round(x)) < margin:
            return False
    return True


@pytest.mark.parametrize("seed", range(4))
def test_weight_table_parity(D, seed):
    B, S = 3, 3000
    r = G.rng(seed, 21)
    toks = np.stack([G.tokens(seed * 10 + b, S) for b in range(B)])
    s = r.standard_normal((B, S)).astype(np.float32)
    s[r.random((B, S)) < 0.2] = np.nan
    if seed == 3:
        toks[2] = 7                      # no delimiter at all -> all zeros
    for b in range(B):
        assert _table_certified(toks[b], s[b], G.T7_IDS)
    w10 = D.weight_table(t(toks), t(G.T7_IDS), t(s)).cpu().numpy()
    for b in range(B):
        ref, _ = O.weight_table(toks[b], s[b], G.T7_IDS)
        assert w10[b].tolist() == ref.tolist()


@pytest.mark.parametrize("S,n_ids", [(3 * 4096 + 123, 13), (2 * 4096, 13), (9000, 64), (131072, 13)])
def test_weight_table_parity_tiles(D, S, n_ids):
    """Several 4096-position smem tiles plus a ragged tail; 64 ids (the API
    maximum: the largest shared-memory footprint); the 128K C5 length."""
    B = 2
    r = G.rng(S + n_ids, 22)
    if n_ids == 13:
        ids = G.T7_IDS
        toks = np.stack([G.tokens(S + b, S) for b in range(B)])
    else:
        ids = np.arange(1000, 1000 + n_ids, dtype=np.int32)
        toks = r.integers(900, 1000 + n_ids + 100, size=(B, S)).astype(np.int32)
    for tries in range(20):
        s = r.standard_normal((B, S)).astype(np.float32)
        s[r.random((B, S)) < 0.1] = np.nan
        if all(_table_certified(toks[b], s[b], ids) for b in range(B)):
            break
    else:
        pytest.fail("no certified table")
    w10 = D.weight_table(t(toks), t(ids), t(s)).cpu().numpy()
    for b in range(B):
        ref, _ = O.weight_table(toks[b], s[b], ids)
        assert w10[b].tolist() == ref.tolist()


# ---------------------------------------------------------------- a4 map + repack + digest
@pytest.mark.parametrize("dtype,P,S", [("bf16", 16, 4099), ("fp32", 16, 2000), ("bf16", 8, 1500),
                                       ("bf16", 32, 777), ("bf16", 16, 1)])
def test_map_repack_digest_parity(D, dtype, P, S):
    B, Hkv, d = 2, 4, 128
    cfg = D.default_config(page_size=P)
    toks = np.stack([G.tokens(200 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    _, K0, V0 = G.decode_qkv(7, S, Hkv, Hkv, d, dtype=dtype)
    K = np.stack([K0, K0[::-1]])
    V = np.stack([V0, -V0])
    layer = D.build_blocks(t(toks), t(G.T7_IDS), t(K, kv_dtype(dtype)), t(V, kv_dtype(dtype)), cfg,
                           static_w10=G.T7_W10, Hq=Hkv)
    torch.cuda.synchronize()
    mb, mp = D.max_blocks(S, cfg), D.max_pages(S, cfg)
    for b in range(B):
        nb = int(layer.n_blocks[b])
        assert layer.block_starts[b, : nb + 1].tolist() == starts[b]
        pf, pb, pv = O.page_map(starts[b], P)
        npg = int(pf[-1])
        assert int(layer.n_pages[b]) == npg
        assert layer.page_first[b, : nb + 1].tolist() == pf.tolist()
        assert np.all(layer.page_first[b, nb + 1:].cpu().numpy() == npg)
        assert layer.page_block[b, :npg].tolist() == pb.tolist()
        assert layer.page_valid[b, :npg].tolist() == pv.tolist()
        assert np.all(layer.page_block[b, npg:mp].cpu().numpy() == -1)
        assert np.all(layer.page_valid[b, npg:mp].cpu().numpy() == 0)
        Kp_ref = O.repack(K[b], starts[b], P)          # [H, n_pages, P, d], zero padding
        Vp_ref = O.repack(V[b], starts[b], P)
        assert np.array_equal(layer.Kp[b, :, :npg].float().cpu().numpy(), Kp_ref)
        assert np.array_equal(layer.Vp[b, :, :npg].float().cpu().numpy(), Vp_ref)
        kmax, kmin = O.digests(K[b], starts[b])
        dig = layer.digests[b, :, :nb].float().cpu().numpy()
        assert np.array_equal(dig[:, :, 0], kmax) and np.array_equal(dig[:, :, 1], kmin)


# ---------------------------------------------------------------- a5 + a6 selection
def _build(D, toks, K, V, cfg, dtype, Hq):
    return D.build_blocks(t(toks), t(G.T7_IDS), t(K, kv_dtype(dtype)), t(V, kv_dtype(dtype)), cfg,
                          static_w10=G.T7_W10, Hq=Hq)


def _check_selection(layer, sel, res, B, Hq):
    ns = sel.n_sel.cpu().numpy()
    sb = sel.sel_blocks.cpu().numpy()
    mg = sel.marginal_block.cpu().numpy()
    kp = sel.marginal_keep.cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            assert sb[b, h, : ns[b, h]].tolist() == res[b]["sel_blocks"][h], (b, h)
            assert (int(mg[b, h]), int(kp[b, h])) == (res[b]["marginal"][h], res[b]["keep"][h]), (b, h)


@pytest.mark.parametrize("Hq,Hkv", [(8, 8), (16, 8), (32, 8), (16, 2)])
def test_select_regime_A_exact(D, Hq, Hkv):
    # integer q, K: every fp32 block score is exact -> frequent ties exercise
    # the (score desc, index asc) rule bit-exactly.
    B, S, d, budget = 2, 3000, 128, 300
    cfg = D.default_config()
    toks = np.stack([G.tokens(300 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv_integer(400 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    layer = _build(D, toks, K, V, cfg, "bf16", Hq)
    sel = D.select(t(q, torch.bfloat16), layer, budget)
    torch.cuda.synchronize()
    res = H.oracle_decode(q, K, V, starts, budget)
    sc = sel.scores.cpu().numpy()
    n_ties = 0
    for b in range(B):
        nb = len(starts[b]) - 1
        for h in range(Hq):
            assert np.array_equal(sc[b, h, :nb].astype(np.float64), res[b]["scores"][h])
            n_ties += nb - len(np.unique(res[b]["scores"][h]))
    assert n_ties > 0
    _check_selection(layer, sel, res, B, Hq)


@pytest.mark.parametrize("dtype,S,Hq,Hkv,budget", [("bf16", 8192, 32, 8, 1024),
                                                   ("fp32", 4096, 8, 8, 512),
                                                   ("bf16", 5000, 16, 2, 777),
                                                   ("bf16", 3000, 8, 1, 16)])
def test_select_regime_B_certified(D, dtype, S, Hq, Hkv, budget):
    B, d = 2, 128
    cfg = D.default_config()
    toks = np.stack([G.tokens(500 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(600 + b, S, Hq, Hkv, d, dtype=dtype) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    q = H.certify_queries(600, q, K, starts, budget, dtype)
    layer = _build(D, toks, K, V, cfg, dtype, Hq)
    sel = D.select(t(q, kv_dtype(dtype)), layer, budget)
    torch.cuda.synchronize()
    res = H.oracle_decode(q, K, V, starts, budget)
    sc = sel.scores.cpu().numpy()
    for b in range(B):
        nb = len(starts[b]) - 1
        kmax, kmin = O.digests(K[b], starts[b])
        for h in range(Hq):
            eps = H.score_error_bound(q[b, h], kmax[h // (Hq // Hkv)], kmin[h // (Hq // Hkv)], dtype == "bf16")
            assert np.all(np.abs(sc[b, h, :nb] - res[b]["scores"][h]) <= eps + 1e-30)
    _check_selection(layer, sel, res, B, Hq)


@pytest.mark.parametrize("S,Hq,Hkv,budget,integer", [(8192, 32, 8, 1024, False), (3000, 16, 2, 300, True),
                                                      (5000, 8, 8, 640, False), (2500, 64, 8, 200, True)])
def test_score_kernels_agree(D, S, Hq, Hkv, budget, integer):
    """a5 on the tensor cores (k_score_blocks_tc, the bf16 default) and the
    CUDA-core half-warp kernel (test hook): both within the score bound of the
    oracle (exactly equal to it for integer q, K), and the same selection."""
    import ctypes
    B, d = 2, 128
    cfg = D.default_config()
    toks = np.stack([G.tokens(1900 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    gen = G.decode_qkv_integer if integer else G.decode_qkv
    qs, Ks, Vs = zip(*[gen(1910 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    if not integer:
        q = H.certify_queries(1910, q, K, starts, budget, "bf16")
    layer = _build(D, toks, K, V, cfg, "bf16", Hq)
    lib = D.lib()
    lib.dynsplit_debug_a5_cuda_core.argtypes = [ctypes.c_int]
    sels = []
    try:
        for cc in (0, 1):
            lib.dynsplit_debug_a5_cuda_core(cc)
            sels.append(D.select(t(q, torch.bfloat16), layer, budget))
            torch.cuda.synchronize()
    finally:
        lib.dynsplit_debug_a5_cuda_core(0)
    res = H.oracle_decode(q, K, V, starts, budget)
    for sel in sels:
        sc = sel.scores.cpu().numpy()
        for b in range(B):
            nb = len(starts[b]) - 1
            kmax, kmin = O.digests(K[b], starts[b])
            for h in range(Hq):
                if integer:
                    assert np.array_equal(sc[b, h, :nb].astype(np.float64), res[b]["scores"][h])
                else:
                    eps = H.score_error_bound(q[b, h], kmax[h // (Hq // Hkv)], kmin[h // (Hq // Hkv)], True)
                    assert np.all(np.abs(sc[b, h, :nb] - res[b]["scores"][h]) <= eps + 1e-30)
        _check_selection(layer, sel, res, B, Hq)
    for name in ("n_sel", "marginal_block", "marginal_keep"):
        assert torch.equal(getattr(sels[0], name), getattr(sels[1], name)), name
    ns = sels[0].n_sel.cpu().numpy()
    s0, s1 = sels[0].sel_blocks.cpu().numpy(), sels[1].sel_blocks.cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            assert np.array_equal(s0[b, h, :ns[b, h]], s1[b, h, :ns[b, h]]), (b, h)


@pytest.mark.parametrize("cuda_core", [0, 1])
def test_short_blocks_score_rounds(D, cuda_core):
    """A plan of minimum-length blocks (C - Delta = 18 tokens everywhere, the
    shortest DD-Select can emit) has more blocks than the launchers expect
    (1.25 S / C): the tensor-core a5 runs its staging rounds, the CUDA-core a5
    its beyond-the-stage global loads.  Integer q, K: scores exact; selection
    and attention against the oracle on the same plan."""
    import ctypes
    B, S, Hq, Hkv, d, budget = 2, 20000, 32, 8, 128, 1500
    cfg = D.default_config()
    L = cfg.C - cfg.delta
    starts = list(range(0, S, L)) + [S]
    assert len(starts) - 1 > 1.25 * S / cfg.C
    qs, Ks, Vs = zip(*[G.decode_qkv_integer(1950 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    toks = np.stack([G.tokens(1960 + b, S) for b in range(B)])
    base = _build(D, toks, K, V, cfg, "bf16", Hq)          # shapes, w10
    mb = D.max_blocks(S, cfg)
    bs = torch.full((B, mb + 1), S, dtype=torch.int32)
    bs[:, : len(starts)] = torch.tensor(starts, dtype=torch.int32)
    bs = bs.cuda()
    nb = torch.full((B,), len(starts) - 1, dtype=torch.int32, device="cuda")
    pf, pb, pv, npg = D.map_pages(bs, nb, S, cfg)
    Kp, Vp, dig = D.repack_digest(t(K, torch.bfloat16), t(V, torch.bfloat16), bs, nb, pf, cfg)
    layer = D.PagedLayer(base.shape, cfg, base.w10, bs, nb, pf, pb, pv, npg, Kp, Vp, dig)
    lib = D.lib()
    lib.dynsplit_debug_a5_cuda_core.argtypes = [ctypes.c_int]
    try:
        lib.dynsplit_debug_a5_cuda_core(cuda_core)
        qt = t(q, torch.bfloat16)
        sel = D.select(qt, layer, budget)
        o, lse = D.decode_attn(qt, layer, sel.worklist)
        torch.cuda.synchronize()
    finally:
        lib.dynsplit_debug_a5_cuda_core(0)
    res = H.oracle_decode(q, K, V, [starts] * B, budget)
    sc = sel.scores.cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            assert np.array_equal(sc[b, h, : len(starts) - 1].astype(np.float64), res[b]["scores"][h]), (b, h)
    _check_selection(layer, sel, res, B, Hq)
    _check_attention(o, lse, res, B, Hq)


# ---------------------------------------------------------------- a7 + a8 attention
def _check_attention(o, lse, res, B, Hq):
    o = o.cpu().numpy()
    lse = lse.cpu().numpy()
    worst = 0.0
    for b in range(B):
        err = H.row_rel_err(o[b], res[b]["o"])
        worst = max(worst, float(err.max()))
        assert np.all(err <= ATT_TOL), err.max()
        assert np.all(np.abs(lse[b] - res[b]["lse"]) <= LSE_TOL * np.maximum(1, np.abs(res[b]["lse"])))
    return worst


@pytest.mark.parametrize("dtype,S,Hq,Hkv,budget,rho", [
    ("fp32", 4096, 8, 8, 512, 0.0),        # C1 shape
    ("bf16", 8192, 32, 8, 2048, 0.0),      # C2 head layout, reduced S
    ("bf16", 8192, 32, 8, 2048, 0.9),
    ("bf16", 6001, 40, 40, 700, 0.0),      # C4 head layout (MHA), ragged
    ("bf16", 4000, 64, 8, 333, 0.5),       # g = 8
    ("bf16", 2000, 8, 4, 5000, 0.0),       # budget >= S -> dense
    ("bf16", 2000, 8, 4, 1, 0.0),          # budget 1
    ("bf16", 1, 8, 2, 1, 0.0),             # a single token: one block, one page
    ("bf16", 17, 32, 8, 5, 0.0),           # one partial block
    ("bf16", 47, 8, 2, 20, 0.0),           # two blocks, ragged page tail
    ("fp32", 50, 8, 8, 20, 0.0),
])
def test_sparse_decode_parity(D, dtype, S, Hq, Hkv, budget, rho):
    B, d = 2, 128
    cfg = D.default_config()
    toks = np.stack([G.tokens(700 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(800 + b, S, Hq, Hkv, d, rho=rho, dtype=dtype) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    q = H.certify_queries(800, q, K, starts, budget, dtype)
    layer = _build(D, toks, K, V, cfg, dtype, Hq)
    qt = t(q, kv_dtype(dtype))
    sel = D.select(qt, layer, budget)
    o, lse = D.decode_attn(qt, layer, sel.worklist)
    torch.cuda.synchronize()
    res = H.oracle_decode(q, K, V, starts, budget)
    _check_selection(layer, sel, res, B, Hq)
    _check_attention(o, lse, res, B, Hq)
    # repeat (workspace counters must be left zeroed) -> identical bits
    o2, lse2 = D.decode_attn(qt, layer, sel.worklist)
    assert torch.equal(o, o2) and torch.equal(lse, lse2)


@pytest.mark.parametrize("dtype,S,Hq,Hkv", [("bf16", 5000, 32, 8), ("fp32", 4096, 8, 8), ("bf16", 700, 4, 4)])
def test_dense_decode_parity(D, dtype, S, Hq, Hkv):
    B, d = 2, 128
    cfg = D.default_config()
    toks = np.stack([G.tokens(900 + b, S) for b in range(B)])
    qs, Ks, Vs = zip(*[G.decode_qkv(950 + b, S, Hq, Hkv, d, dtype=dtype) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    layer = _build(D, toks, K, V, cfg, dtype, Hq)
    o, lse = D.decode_attn(t(q, kv_dtype(dtype)), layer, None)
    torch.cuda.synchronize()
    g = Hq // Hkv
    res = []
    for b in range(B):
        oo = np.zeros((Hq, d))
        ll = np.zeros(Hq)
        for h in range(Hq):
            oo[h], ll[h] = O.dense_attention(q[b, h], K[b, :, h // g], V[b, :, h // g], 1 / math.sqrt(d))
        res.append({"o": oo, "lse": ll})
    _check_attention(o, lse, res, B, Hq)


def test_merge_partials_parity(D):
    r = G.rng(3, 31)
    n, rows, d = 5, 7, 128
    o_parts = r.standard_normal((n, rows, d)).astype(np.float32)
    lse_parts = r.standard_normal((n, rows)).astype(np.float32) * 3
    lse_parts[1, 2] = -np.inf
    lse_parts[:, 4] = -np.inf                      # a row no part saw
    o, lse = D.merge_partials(t(o_parts), t(lse_parts))
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    for i in range(rows):
        ro, rl = O.merge_partials(o_parts[:, i], lse_parts[:, i])
        if rl == -np.inf:
            assert lse[i] == -np.inf and np.all(o[i] == 0)
        else:
            assert H.row_rel_err(o[i], ro) <= 1e-5 and abs(lse[i] - rl) <= 1e-5


def test_decode_step_host_matches_device_path(D):
    B, S, Hq, Hkv, d, budget = 2, 4000, 32, 8, 128, 512
    cfg = D.default_config()
    toks = np.stack([G.tokens(1000 + b, S) for b in range(B)])
    qs, Ks, Vs = zip(*[G.decode_qkv(1100 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    layer = _build(D, toks, K, V, cfg, "bf16", Hq)
    qt = t(q, torch.bfloat16)
    sel = D.select(qt, layer, budget)
    o_ref, lse_ref = D.decode_attn(qt, layer, sel.worklist)
    shape = D.make_shape(B, S, Hq, Hkv)
    ws = torch.zeros(D.step_host_workspace_bytes(shape, cfg, budget), dtype=torch.uint8, device=DEV)
    wl = torch.empty(D.worklist_bytes(shape, cfg, budget), dtype=torch.uint8, device=DEV)
    qh = qt.cpu().pin_memory()
    oh = torch.empty(B, Hq, d, dtype=torch.float32).pin_memory()
    lh = torch.empty(B, Hq, dtype=torch.float32).pin_memory()
    D.decode_step_host(qh, layer, budget, oh, lh, wl, ws)
    torch.cuda.synchronize()
    assert torch.equal(oh, o_ref.cpu()) and torch.equal(lh, lse_ref.cpu())


# ---------------------------------------------------------------- a1 scoring + dynamic build
def _score_case(seed, Ls, B, S, Hq, Hkv):
    toks = np.stack([G.tokens(seed + b, S) for b in range(B)])
    Qs, Ks = zip(*[G.scoring_qk(seed + 50 + b, Ls, S, Hq, Hkv) for b in range(B)])
    Qs = np.stack(Qs, axis=1)         # [Ls, B, S, Hq, d]
    Ks = np.stack(Ks, axis=1)
    return toks, Qs, Ks


@pytest.mark.parametrize("kernel", ["tcgen05", "mma.sync"])
@pytest.mark.parametrize("Ls,B,S,Hq,Hkv,R", [(1, 1, 700, 4, 4, 128), (2, 2, 1500, 8, 2, 128),
                                             (1, 1, 333, 2, 1, 16), (1, 2, 1100, 4, 2, 300),
                                             (1, 1, 129, 8, 8, 128)])
def test_score_delimiters_parity(D, Ls, B, S, Hq, Hkv, R, kernel):
    """a1 through both kernels: k_lse_band_tc (tcgen05, the default) and the
    mma.sync k_lse_band (test hook), each within 2e-4 of the oracle."""
    import ctypes
    cfg = D.default_config(R=R)
    toks, Qs, Ks = _score_case(1200, Ls, B, S, Hq, Hkv)
    lib = D.lib()
    lib.dynsplit_debug_a1_mmasync.argtypes = [ctypes.c_int]
    try:
        lib.dynsplit_debug_a1_mmasync(1 if kernel == "mma.sync" else 0)
        s = D.score_delimiters(t(toks), t(G.T7_IDS), t(Qs, torch.bfloat16), t(Ks, torch.bfloat16), cfg)
        s = s.cpu().numpy()
    finally:
        lib.dynsplit_debug_a1_mmasync(0)
    worst = 0.0
    for b in range(B):
        ref = O.score_delimiters(toks[b], G.T7_IDS, Qs[:, b], Ks[:, b], cfg.W, R, cfg.alpha_pen)
        nan_ref = np.isnan(ref)
        assert np.array_equal(np.isnan(s[b]), nan_ref)
        err = np.abs(s[b][~nan_ref] - ref[~nan_ref])
        worst = max(worst, float(err.max()))
        assert np.all(err <= 2e-4), err.max()


def test_dynamic_build_blocks_parity(D):
    # a1 -> a2 -> a3 -> a4 in one C call, vs the oracle pipeline; the seed is
    # chosen so that the oracle's table is margin-certified (P2 rounding).
    B, S, Hq, Hkv, d = 2, 1500, 8, 2, 128
    cfg = D.default_config()
    for seed in range(1300, 1330):
        toks, Qs, Ks = _score_case(seed, 1, B, S, Hq, Hkv)
        sref = [O.score_delimiters(toks[b], G.T7_IDS, Qs[:, b], Ks[:, b]) for b in range(B)]
        if all(_table_certified(toks[b], sref[b], G.T7_IDS, margin=1e-2) for b in range(B)):
            break
    else:
        pytest.fail("no certified seed")
    _, K0, V0 = G.decode_qkv(seed, S, Hkv, Hkv, d)
    K = np.stack([K0, K0[::-1]])
    V = np.stack([V0, V0[::-1]])
    layer = D.build_blocks(t(toks), t(G.T7_IDS), t(K, torch.bfloat16), t(V, torch.bfloat16), cfg,
                           Qs=t(Qs, torch.bfloat16), Ks=t(Ks, torch.bfloat16), return_scores=True)
    torch.cuda.synchronize()
    for b in range(B):
        w_ref, _ = O.weight_table(toks[b], sref[b], G.T7_IDS)
        assert layer.w10[b].tolist() == w_ref.tolist()
        st_ref = O.segment(toks[b], G.T7_IDS, w_ref, 32, 14)
        nb = int(layer.n_blocks[b])
        assert layer.block_starts[b, : nb + 1].tolist() == st_ref
        kmax, kmin = O.digests(K[b], st_ref)
        dig = layer.digests[b, :, :nb].float().cpu().numpy()
        assert np.array_equal(dig[:, :, 0], kmax) and np.array_equal(dig[:, :, 1], kmin)


# ---------------------------------------------------------------- the two a6 kernels agree
def _wl_entries(wl, B, Hkv):
    raw = wl.cpu().numpy()
    nbh = B * Hkv
    max_wl = int(raw[:256].view(np.int32)[1])
    counts = raw[256:256 + 4 * nbh].view(np.int32).copy()
    off = 256 + ((4 * nbh + 255) // 256) * 256
    ent = raw[off: off + 16 * nbh * max_wl].reshape(max_wl, nbh, 16)
    return counts, [ent[: counts[i], i].copy() for i in range(nbh)]


@pytest.mark.parametrize("kind,S,Hq,Hkv,budget", [
    ("float", 8192, 32, 8, 1024),      # C3 head layout
    ("int", 3000, 16, 2, 300),         # integer scores: many exact ties
    ("zero", 2500, 8, 4, 200),         # q = 0: every score equal -> index order
    ("float", 1500, 8, 8, 100000),     # everything fits
    ("float", 40, 4, 4, 5),            # a handful of blocks
])
def test_select_kernels_agree(D, kind, S, Hq, Hkv, budget):
    """k_select_reg (register-resident, <= 8192 blocks) and the generic
    k_select produce bit-identical selections, marginals and worklists."""
    import ctypes
    B, d = 2, 128
    cfg = D.default_config()
    toks = np.stack([G.tokens(900 + b, S) for b in range(B)])
    if kind == "int":
        qs, Ks, Vs = zip(*[G.decode_qkv_integer(910 + b, S, Hq, Hkv, d) for b in range(B)])
    else:
        qs, Ks, Vs = zip(*[G.decode_qkv(910 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    if kind == "zero":
        q = np.zeros_like(q)
    layer = _build(D, toks, K, V, cfg, "bf16", Hq)
    qt = t(q, torch.bfloat16)
    lib = D.lib()
    lib.dynsplit_debug_select_generic.argtypes = [ctypes.c_int]
    reg = D.select(qt, layer, budget)
    torch.cuda.synchronize()
    try:
        lib.dynsplit_debug_select_generic(1)
        gen = D.select(qt, layer, budget)
        torch.cuda.synchronize()
    finally:
        lib.dynsplit_debug_select_generic(0)
    for name in ("n_sel", "marginal_block", "marginal_keep"):
        assert torch.equal(getattr(reg, name), getattr(gen, name)), name
    ns = reg.n_sel.cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            assert torch.equal(reg.sel_blocks[b, h, : ns[b, h]], gen.sel_blocks[b, h, : ns[b, h]])
    cf, ef = _wl_entries(reg.worklist, B, Hkv)
    cr, er = _wl_entries(gen.worklist, B, Hkv)
    assert np.array_equal(cf, cr)
    for a, c in zip(ef, er):
        assert np.array_equal(a, c)
    if kind == "zero":   # all scores equal: whole blocks in index order
        for b in range(B):
            st = layer.block_starts[b, : int(layer.n_blocks[b]) + 1].cpu().numpy()
            m = int(np.searchsorted(st, budget - 1, side="right")) - 1
            assert reg.marginal_block[b].tolist() == [m] * Hq
            assert reg.marginal_keep[b].tolist() == [budget - int(st[m])] * Hq


@pytest.mark.parametrize("S,Hq,Hkv,budget", [(8192, 32, 8, 1024), (3000, 8, 2, 5000), (2000, 8, 8, 1)])
def test_decode_layer_matches_separate_calls(D, S, Hq, Hkv, budget):
    """dynsplit_decode_layer (a5-a8 in one call) == dynsplit_select +
    dynsplit_decode_attn bit for bit, and == the oracle."""
    B, d = 2, 128
    cfg = D.default_config()
    toks = np.stack([G.tokens(950 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(960 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    q = H.certify_queries(960, q, K, starts, budget, "bf16")
    layer = _build(D, toks, K, V, cfg, "bf16", Hq)
    qt = t(q, torch.bfloat16)
    o1, lse1, sel1 = D.decode_layer(qt, layer, budget)
    sel2 = D.select(qt, layer, budget)
    o2, lse2 = D.decode_attn(qt, layer, sel2.worklist)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(lse1, lse2)
    for name in ("n_sel", "marginal_block", "marginal_keep"):
        assert torch.equal(getattr(sel1, name), getattr(sel2, name)), name
    res = H.oracle_decode(q, K, V, starts, budget)
    _check_attention(o1, lse1, res, B, Hq)


@pytest.mark.parametrize("B,S,Hq,Hkv,budget", [(8, 3000, 32, 8, 400), (16, 1500, 8, 2, 200)])
def test_decode_large_batch(D, B, S, Hq, Hkv, budget):
    """Many sequences per launch: few attention splits per (b, KV head), a5 /
    a6 grids over B * Hkv, ragged block counts across the batch; through
    dynsplit_decode_layer, against the oracle."""
    d = 128
    cfg = D.default_config()
    toks = np.stack([G.tokens(1500 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(1600 + b, S, Hq, Hkv, d) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    q = H.certify_queries(1600, q, K, starts, budget, "bf16")
    layer = _build(D, toks, K, V, cfg, "bf16", Hq)
    qt = t(q, torch.bfloat16)
    o, lse, sel_l = D.decode_layer(qt, layer, budget)
    sel = D.select(qt, layer, budget)
    torch.cuda.synchronize()
    res = H.oracle_decode(q, K, V, starts, budget)
    _check_selection(layer, sel, res, B, Hq)
    assert torch.equal(sel_l.n_sel, sel.n_sel)
    _check_attention(o, lse, res, B, Hq)


def test_decode_layers_back_to_back_shared_buffers(D):
    """Many layers through dynsplit_decode_layer back to back on ONE
    workspace and ONE worklist buffer (as the e2e step does), PDL-chained,
    eagerly and as a replayed CUDA graph: every layer equals its isolated,
    synchronised call bit for bit (no stale worklist / score reads across
    layers), and the oracle."""
    B, S, Hq, Hkv, d, L, budget = 2, 12000, 32, 8, 128, 6, 1000
    cfg = D.default_config()
    toks = np.stack([G.tokens(1400 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    layers, qs, host = [], [], []
    for l in range(L):
        qkv = [G.decode_qkv(1410 + 10 * l + b, S, Hq, Hkv, d) for b in range(B)]
        q, K, V = (np.stack(x) for x in zip(*qkv))
        q = H.certify_queries(1410 + 10 * l, q, K, starts, budget, "bf16")
        layers.append(_build(D, toks, K, V, cfg, "bf16", Hq))
        qs.append(t(q, torch.bfloat16))
        host.append((q, K, V))
    ref = []
    for l in range(L):                                     # isolated calls
        o, lse, sel = D.decode_layer(qs[l], layers[l], budget)
        torch.cuda.synchronize()
        ref.append((o.clone(), lse.clone(), sel.n_sel.clone()))
    shape = D._decode_shape(qs[0], layers[0])
    ws = torch.zeros(D.workspace_bytes(D.OP_DECODE_LAYER, shape, cfg, budget), dtype=torch.uint8, device="cuda")
    _, ns, mg, kp, wl = D._sel_outputs(shape, cfg, budget, qs[0].device, want_blocks=False)
    outs = [(torch.empty(B, Hq, d, device="cuda"), torch.empty(B, Hq, device="cuda")) for _ in range(L)]
    nsl = [torch.empty_like(ns) for _ in range(L)]

    def run_all():
        for l in range(L):
            D.decode_layer(qs[l], layers[l], budget, out=(nsl[l], mg, kp, wl, outs[l][0], outs[l][1]), ws=ws)

    def check():
        for l in range(L):
            assert torch.equal(outs[l][0], ref[l][0]) and torch.equal(outs[l][1], ref[l][1]), l
            assert torch.equal(nsl[l], ref[l][2]), l

    for _ in range(3):
        run_all()
    torch.cuda.synchronize()
    check()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        run_all()
    torch.cuda.current_stream().wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run_all()
    for _ in range(4):
        for o in outs:
            o[0].fill_(float("nan"))
        g.replay()
    torch.cuda.synchronize()
    check()
    for l in (0, L - 1):
        q, K, V = host[l]
        res = H.oracle_decode(q, K, V, starts, budget)
        _check_attention(outs[l][0], outs[l][1], res, B, Hq)


# ---------------------------------------------------------------- NEXT-2: mean-pooling digests
@pytest.mark.parametrize("dtype,S,Hq,Hkv,budget", [("bf16", 6000, 32, 8, 900), ("fp32", 3000, 8, 8, 400),
                                                   ("bf16", 4000, 16, 2, 5000)])
def test_mean_mode_parity(D, dtype, S, Hq, Hkv, budget):
    """digest_mode = 1: the fp32 block means within their
    rounding bound, the selection exactly (margin-certified queries) and the
    attention within 2e-3, against the oracle's mean-pooling decode step."""
    B, d = 2, 128
    cfg = D.default_config(digest_mode=1)
    toks = np.stack([G.tokens(1700 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(1710 + b, S, Hq, Hkv, d, dtype=dtype) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    q = H.certify_queries_mean(1710, q, K, starts, budget, dtype)
    layer = _build(D, toks, K, V, cfg, dtype, Hq)
    qt = t(q, kv_dtype(dtype))
    sel = D.select(qt, layer, budget)
    o, lse = D.decode_attn(qt, layer, sel.worklist)
    torch.cuda.synchronize()
    mb = D.max_blocks(S, cfg)
    dig = layer.digests.contiguous().view(torch.float32).reshape(B, Hkv, mb, -1)[..., :d].cpu().numpy()
    for b in range(B):
        nb = len(starts[b]) - 1
        km = O.digests_mean(K[b], starts[b])
        assert np.all(np.abs(dig[b, :, :nb] - km) <= H.mean_digest_error_bound(K[b], starts[b]))
    res = [O.decode_step(q[b], K[b], V[b], starts[b], budget, digest_mode="mean") for b in range(B)]
    _check_selection(layer, sel, res, B, Hq)
    _check_attention(o, lse, res, B, Hq)


@pytest.mark.parametrize("S,Hq,Hkv,budget,rho", [(8192, 32, 8, 2048, 0.0), (6001, 40, 40, 700, 0.0),
                                                 (4000, 64, 8, 333, 0.5), (47, 8, 2, 20, 0.0)])
def test_sparse_decode_parity_tma_variant(D, monkeypatch, S, Hq, Hkv, budget, rho):
    """The A/B variant of k_decode_attn whose pages move by 2-D TMA boxes
    (DYNSPLIT_ATTN_TMA=1; measured slower): same selection,
    attention against the oracle, and the sparse / dense results equal to the
    LDGSTS kernel up to fp32 rounding (same page order, same arithmetic)."""
    B, d, dtype = 2, 128, "bf16"
    cfg = D.default_config()
    toks = np.stack([G.tokens(1700 + b, S) for b in range(B)])
    starts = [O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    qs, Ks, Vs = zip(*[G.decode_qkv(1800 + b, S, Hq, Hkv, d, rho=rho, dtype=dtype) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    q = H.certify_queries(1800, q, K, starts, budget, dtype)
    layer = _build(D, toks, K, V, cfg, dtype, Hq)
    qt = t(q, kv_dtype(dtype))
    sel = D.select(qt, layer, budget)
    o_l, lse_l = D.decode_attn(qt, layer, sel.worklist)
    od_l, lsed_l = D.decode_attn(qt, layer, None)
    monkeypatch.setenv("DYNSPLIT_ATTN_TMA", "1")
    o, lse = D.decode_attn(qt, layer, sel.worklist)
    od, lsed = D.decode_attn(qt, layer, None)
    torch.cuda.synchronize()
    monkeypatch.delenv("DYNSPLIT_ATTN_TMA")
    res = H.oracle_decode(q, K, V, starts, budget)
    _check_attention(o, lse, res, B, Hq)
    for a, b_ in ((o, o_l), (od, od_l)):
        assert np.all(H.row_rel_err(a.cpu().numpy().reshape(-1, d), b_.cpu().numpy().reshape(-1, d)) <= 1e-5)
    assert torch.allclose(lse, lse_l, rtol=0, atol=1e-5) and torch.allclose(lsed, lsed_l, rtol=0, atol=1e-5)

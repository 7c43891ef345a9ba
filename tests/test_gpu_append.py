"""NEXT-1 parity: decode-time append with incremental DD-Select
(dynsplit_append_plan / dynsplit_append_kv) against the oracle on the grown
sequence.  A prefix is planned and paged through the append path
(L_prev = 0), then tokens arrive one at a time (and once several at a time);
at checkpoints the plan, page tables, pages and digests must equal
segment / page_map / repack / digests of the oracle on the whole prefix
(bit-exact), and a decode step on the grown cache must match the oracle."""
import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G
from tests import helpers as H

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def t(x, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(x)).to(DEV, dtype=dtype)


def _check_layer(layer, toks, K, V, L, C, delta, P, Hkv, mean=False):
    B = toks.shape[0]
    for b in range(B):
        starts = O.segment(toks[b, :L], G.T7_IDS, G.T7_W10, C, delta)
        nb = len(starts) - 1
        assert int(layer.n_blocks[b]) == nb
        assert layer.block_starts[b, : nb + 1].tolist() == starts
        pf, pb, pv = O.page_map(starts, P)
        npg = int(pf[-1])
        assert int(layer.n_pages[b]) == npg
        assert layer.page_first[b, : nb + 1].tolist() == pf.tolist()
        assert layer.page_block[b, :npg].tolist() == pb.tolist()
        assert layer.page_valid[b, :npg].tolist() == pv.tolist()
        kp = layer.Kp[b, :, :npg].float().cpu().numpy()
        vp = layer.Vp[b, :, :npg].float().cpu().numpy()
        assert np.array_equal(kp, O.repack(K[b, :L], starts, P))
        assert np.array_equal(vp, O.repack(V[b, :L], starts, P))
        if mean:  # NEXT-2 mean pooling: fp32 means within their rounding bound
            dig = layer.digests[b].contiguous().view(torch.float32)
            dig = dig.reshape(dig.shape[0], dig.shape[1], -1)[:, :nb, :128].cpu().numpy()
            assert np.all(np.abs(dig - O.digests_mean(K[b, :L], starts)) <=
                          H.mean_digest_error_bound(K[b, :L], starts))
        else:
            kmax, kmin = O.digests(K[b, :L], starts)
            dig = layer.digests[b, :, :nb].float().cpu().numpy()
            assert np.array_equal(dig[:, :, 0], kmax) and np.array_equal(dig[:, :, 1], kmin)
    return starts


@pytest.mark.parametrize("dtype,C,delta,P,S0,steps,multi", [
    ("bf16", 32, 14, 16, 700, 40, 5),
    ("fp32", 16, 5, 8, 300, 30, 3),
    ("bf16", 32, 14, 16, 1, 60, 0),      # from a single token
    ("bf16", 64, 14, 32, 500, 20, 70),   # a multi-token step longer than C + Delta
    ("bf16-mean", 32, 14, 16, 400, 25, 4),  # mean-pooling digests (NEXT-2)
])
def test_append_matches_oracle(dtype, C, delta, P, S0, steps, multi):
    from paper_2602_03184_b200 import dynsplit as D
    mean = dtype.endswith("-mean")
    dtype = dtype.replace("-mean", "")
    B, Hq, Hkv, d = 2, 4, 2, 128
    S_cap = S0 + steps + multi + 8
    cfg = D.default_config(C=C, delta=delta, page_size=P, digest_mode=int(mean))
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    toks = np.stack([G.tokens(1500 + b, S_cap) for b in range(B)])
    qs, Ks, Vs = zip(*[G.decode_qkv(1510 + b, S_cap, Hq, Hkv, d, dtype=dtype) for b in range(B)])
    q, K, V = np.stack(qs), np.stack(Ks), np.stack(Vs)
    toks_d = t(toks)
    ids = t(G.T7_IDS)
    w10 = t(np.tile(G.T7_W10, (B, 1)), torch.uint8)
    Kd, Vd = t(K, tdt), t(V, tdt)
    lay0 = D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, tdt, DEV)
    lay1 = D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, tdt, DEV, plan_from=lay0)
    ws = D.append_workspace(lay0)

    def step(Lp, L):
        D.append_plan(toks_d, ids, lay0, Lp, L, ws)
        kn, vn = Kd[:, Lp:L].contiguous(), Vd[:, Lp:L].contiguous()
        if (L - Lp) % 2:   # one call per layer ...
            D.append_kv(lay0, kn, vn, Lp, L, ws)
            # a second layer sharing the plan: V and K swapped (independent data)
            D.append_kv(lay1, vn, kn, Lp, L, ws)
        else:              # ... or both layers in one launch
            D.append_kv_layers([lay0, lay1], [kn, vn], [vn, kn], Lp, L, ws)

    step(0, S0)
    torch.cuda.synchronize()
    _check_layer(lay0, toks, K, V, S0, C, delta, P, Hkv, mean)
    L = S0
    for i in range(steps):
        step(L, L + 1)
        L += 1
        if i % 10 == 9:
            torch.cuda.synchronize()
            _check_layer(lay0, toks, K, V, L, C, delta, P, Hkv, mean)
    if multi:
        step(L, L + multi)
        L += multi
    torch.cuda.synchronize()
    starts = _check_layer(lay0, toks, K, V, L, C, delta, P, Hkv, mean)
    _check_layer(lay1, toks, V, K, L, C, delta, P, Hkv, mean)
    # the incremental chain equals the oracle's incremental update too
    prev = O.segment(toks[B - 1, :L - 1], G.T7_IDS, G.T7_W10, C, delta)
    assert O.segment_incremental(prev, toks[B - 1, :L], G.T7_IDS, G.T7_W10, C, delta)[0] == starts

    # a decode step on the grown cache (capacity shape, L valid tokens)
    budget = max(1, L // 4)
    certify = H.certify_queries_mean if mean else H.certify_queries
    qc = certify(1510, q, K[:, :L], [O.segment(toks[b, :L], G.T7_IDS, G.T7_W10, C, delta)
                                     for b in range(B)], budget, dtype)
    qt = t(qc, tdt)
    sel = D.select(qt, lay0, budget)
    o, lse = D.decode_attn(qt, lay0, sel.worklist)
    torch.cuda.synchronize()
    for b in range(B):
        st = O.segment(toks[b, :L], G.T7_IDS, G.T7_W10, C, delta)
        res = O.decode_step(qc[b], K[b, :L], V[b, :L], st, budget, digest_mode="mean" if mean else "minmax")
        ns = sel.n_sel.cpu().numpy()[b]
        sb = sel.sel_blocks.cpu().numpy()[b]
        for h in range(Hq):
            assert sb[h, : ns[h]].tolist() == res["sel_blocks"][h]
        err = H.row_rel_err(o[b].cpu().numpy(), res["o"])
        assert np.all(err <= 2e-3), err.max()

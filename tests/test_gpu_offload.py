"""NEXT-3 parity: host-offloaded KV with cross-step reuse (Appendix B.2
"KVCache Reuse with V2F" Steps 1-3; the CPU-GPU deployment,
P:465-473) through dynsplit_decode_layer_offload /
dynsplit_reuse_plan / dynsplit_fetch_pages, against the oracle's
offload_decode_loop (plan_reuse over the KV heads' page sets).

Over a walk of consecutive decode queries (synth.decode_query_walk) every
step must give, bit-exact: the KV heads' page sets, the fresh (moved) pages,
the reused count, reuse_len, the cache's slot tags (exactly this step's
pages) and the cache rows (equal to the pages they hold); o and lse equal the
resident path on the same worklist bit for bit and the oracle within
the R17 tolerances."""
import ctypes

import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from paper_2602_03184_b200 import dynsplit as D
from synth import generators as G
from tests import helpers as H

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
LSE_TOL = 1e-4


def t(x, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(x)).to(DEV, dtype=dtype)


def _setup(seed, S, Hq, Hkv, budget, T, tau=0.9):
    toks = G.tokens(seed, S)
    q0, K, V = G.decode_qkv(seed + 1, S, Hq, Hkv)
    cfg = D.default_config()
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, cfg.C, cfg.delta)
    qs = G.decode_query_walk(seed + 2, T, q0, tau)
    qs = np.stack([H.certify_queries(seed + 3 + i, qs[i][None], K[None], [starts], budget)[0]
                   for i in range(T)])
    layer = D.build_blocks(t(toks[None]), t(G.T7_IDS), t(K[None], torch.bfloat16), t(V[None], torch.bfloat16),
                           cfg, static_w10=G.T7_W10, Hq=Hq)
    assert layer.block_starts[0, : len(starts)].tolist() == starts
    return toks, qs, K, V, starts, layer


def _run_loop(qs, layer, budget, Hq, truncate, reuse, n_slots=None):
    off = D.offload_layer(layer, budget, Hq, n_slots=n_slots, keep_device=True)
    shape = D.make_shape(1, layer.shape.S, Hq, layer.shape.Hkv)
    ws = D.workspace(D.workspace_bytes(D.OP_DECODE_OFFLOAD, shape, layer.cfg, budget), DEV, "offload_test")
    D.clear_device_error(ws)
    steps = []
    for q in qs:
        qt = t(q[None], torch.bfloat16)
        o, lse, sel = D.decode_layer_offload(qt, off, budget, truncate=truncate, reuse=reuse, ws=ws)
        o_res, lse_res = D.decode_attn(qt, layer, sel.worklist)   # resident pages, same worklist
        torch.cuda.synchronize()
        steps.append(dict(
            o=o[0].cpu().numpy(), lse=lse[0].cpu().numpy(), same_as_resident=bool(
                torch.equal(o, o_res) and torch.equal(lse, lse_res)),
            pages=D.worklist_pages(sel.worklist, shape), cpages=D.worklist_pages(off.worklist_cache, shape),
            fetch=off.fetch.cpu().numpy().copy(), fcount=off.fetch_count.cpu().numpy().copy(),
            stats=off.reuse_stats.cpu().numpy().copy(), rlen=int(off.reuse_len[0]),
            slot_page=off.slot_page.cpu().numpy().copy(),
            cache_ok=_cache_matches(off, layer)))
    err = D.read_device_error(ws)
    return steps, err


def _cache_matches(off, layer):
    """Every occupied slot holds the valid rows of the page it is tagged with."""
    sp = off.slot_page[0]
    pv = layer.page_valid[0]
    for hk in range(sp.shape[0]):
        occ = (sp[hk] >= 0).nonzero().flatten()
        pg = sp[hk, occ].long()
        rows = pv[pg].long()
        kc, kp = off.Kc[0, hk, occ], layer.Kp[0, hk, pg]
        vc, vp = off.Vc[0, hk, occ], layer.Vp[0, hk, pg]
        mask = (torch.arange(kc.shape[1], device=DEV)[None, :] < rows[:, None])[..., None]
        if not (torch.equal(kc * mask, kp * mask) and torch.equal(vc * mask, vp * mask)):
            return False
    return True


def _check_against_oracle(steps, ref, Hkv, truncate, reuse):
    for s, r in zip(steps, ref):
        for hk in range(Hkv):
            pages = np.sort(s["pages"][hk])
            assert pages.tolist() == r["pages"][hk].tolist()          # the union page set (Q18)
            fc = int(s["fcount"][0, hk])
            fp = s["fetch"][0, hk, :fc]
            assert fp[:, 0].tolist() == r["fresh"][hk].tolist()         # moved = fresh, ascending (Step 2)
            assert len(set(fp[:, 1].tolist())) == fc                   # distinct slots
            assert s["stats"][0, hk].tolist() == [len(r["reused"][hk]), len(r["fresh"][hk])]
            tags = s["slot_page"][0, hk]
            assert np.sort(tags[tags >= 0]).tolist() == r["pages"][hk].tolist()  # cache = this step's pages
            # the cache worklist points every entry at the slot holding its page
            slot_of = {int(p): i for i, p in enumerate(tags) if p >= 0}
            assert s["cpages"][hk].tolist() == [slot_of[int(p)] for p in s["pages"][hk]]
        assert s["rlen"] == (r["reuse_len"] if (truncate and reuse) else -1)
        assert s["cache_ok"]
        assert s["same_as_resident"]
        assert H.row_rel_err(s["o"], r["o"]).max() < 2e-3
        assert np.all(np.abs(s["lse"] - r["lse"]) <= LSE_TOL * np.maximum(1.0, np.abs(r["lse"])))


@pytest.mark.parametrize("truncate", [True, False])
@pytest.mark.parametrize("S,Hq,Hkv,budget", [(3000, 8, 2, 256), (2100, 16, 4, 128),
                                              (1500, 12, 12, 128)])   # > 8 KV heads: two-kernel plan
def test_offload_reuse_matches_oracle(S, Hq, Hkv, budget, truncate):
    T = 6
    toks, qs, K, V, starts, layer = _setup(71, S, Hq, Hkv, budget, T)
    steps, err = _run_loop(qs, layer, budget, Hq, truncate, True)
    assert err == 0
    ref = O.offload_decode_loop(qs, K, V, starts, budget, P=layer.cfg.page_size, truncate=truncate)
    _check_against_oracle(steps, ref, Hkv, truncate, True)
    # the walk's neighbouring steps do overlap: something was reused after step 0
    assert sum(int(s["stats"][0, :, 0].sum()) for s in steps[1:]) > 0
    assert int(steps[0]["stats"][0, :, 0].sum()) == 0


def test_offload_without_reuse_moves_every_page():
    toks, qs, K, V, starts, layer = _setup(72, 3000, 8, 2, 256, 4)
    steps, err = _run_loop(qs, layer, 256, 8, True, False)
    assert err == 0
    ref = O.offload_decode_loop(qs, K, V, starts, 256, P=layer.cfg.page_size, reuse=False)
    _check_against_oracle(steps, ref, 2, True, False)
    for s, r in zip(steps, ref):
        assert s["stats"][0, :, 0].tolist() == [0, 0]


def test_offload_capacity_error():
    toks, qs, K, V, starts, layer = _setup(73, 3000, 8, 2, 256, 1)
    steps, err = _run_loop(qs, layer, 256, 8, True, True, n_slots=8)
    assert err & D.DEVERR_PAGE_CAPACITY


def test_fetch_dense_equals_resident_dense():
    toks, qs, K, V, starts, layer = _setup(74, 2500, 8, 2, 256, 1)
    mp = D.max_pages(layer.shape.S, layer.cfg)
    off = D.offload_layer(layer, 256, 8, n_slots=mp, keep_device=True)
    D.fetch_pages(off, 8, dense=True)
    qt = t(qs[0][None], torch.bfloat16)
    o_c, lse_c = D.decode_attn(qt, D.cache_view(off), None)
    o_r, lse_r = D.decode_attn(qt, layer, None)
    torch.cuda.synchronize()
    assert torch.equal(o_c, o_r) and torch.equal(lse_c, lse_r)
    res = O.decode_step(qs[0], K, V, starts, 10 ** 9)               # budget >= S: dense attention
    assert H.row_rel_err(o_c[0].cpu().numpy(), res["o"]).max() < 2e-3


def test_fetch_rejects_pageable_host_memory():
    toks, qs, K, V, starts, layer = _setup(75, 1500, 8, 2, 128, 1)
    off = D.offload_layer(layer, 128, 8)
    with pytest.raises(D.DynsplitError):
        off.Kh = off.Kh.clone()                                       # not pinned
        D.fetch_pages(off, 8)
    pageable = np.zeros(off.Vh.numel() * 2, np.uint8)
    shape = D.make_shape(1, layer.shape.S, 8, 2)
    c = off.c()
    st = D.lib().dynsplit_fetch_pages(ctypes.byref(shape), ctypes.byref(layer.cfg),
                                      ctypes.c_void_p(pageable.ctypes.data), ctypes.c_void_p(off.Vh.data_ptr()),
                                      ctypes.c_void_p(layer.page_valid.data_ptr()),
                                      ctypes.c_void_p(layer.n_pages.data_ptr()), 0, ctypes.byref(c),
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 1                                                    # DYNSPLIT_ERR_INVALID_ARGUMENT


def test_offload_step_graph_replay():
    """The offloaded layer is graph-capturable: replaying one captured step
    over the walk gives the eager loop's plans and outputs."""
    T, budget, Hq = 5, 256, 8
    toks, qs, K, V, starts, layer = _setup(76, 3000, Hq, 2, budget, T)
    eager, _ = _run_loop(qs, layer, budget, Hq, True, True)
    off = D.offload_layer(layer, budget, Hq)
    shape = D.make_shape(1, layer.shape.S, Hq, 2)
    ws = D.workspace(D.workspace_bytes(D.OP_DECODE_OFFLOAD, shape, layer.cfg, budget), DEV, "offload_graph")
    qbuf = torch.empty(1, Hq, 128, dtype=torch.bfloat16, device=DEV)
    _, ns, mg, kp, wl = D._sel_outputs(shape, layer.cfg, budget, DEV, want_blocks=False)
    o = torch.empty(1, Hq, 128, device=DEV)
    lse = torch.empty(1, Hq, device=DEV)
    out = (ns, mg, kp, wl, o, lse)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        qbuf.copy_(t(qs[0][None], torch.bfloat16))
        D.decode_layer_offload(qbuf, off, budget, out=out, ws=ws)       # warm-up (loads, attributes)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    off.reset()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        D.decode_layer_offload(qbuf, off, budget, out=out, ws=ws)
    off.reset()
    for i in range(T):
        qbuf.copy_(t(qs[i][None], torch.bfloat16))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(o[0].cpu().numpy(), eager[i]["o"])
        assert np.array_equal(off.reuse_stats.cpu().numpy(), eager[i]["stats"])

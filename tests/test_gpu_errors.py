"""The device error word (include/dynsplit.h "DYNSPLIT_DEVERR_*"): data-dependent
errors only the kernels can see are reported in the first int32 of the
caller's workspace, the offending sequence is skipped, and nothing is written
out of bounds.  SPEC names: PlanCoverageMismatch, PlanMismatch.

Also the ordering contract: an append (which ends with dynsplit_stream_fence)
followed immediately -- no host synchronisation -- by the PDL-launched decode
kernels must see the appended pages and digests."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G
from tests import helpers as H

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def D():
    from paper_2602_03184_b200 import dynsplit
    dynsplit.lib()
    return dynsplit


def t(x, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(x)).to(DEV, dtype=dtype)


def _layer(D, S=3000, Hq=8, Hkv=2, seed=3, cfg=None):
    cfg = cfg or D.default_config()
    toks = G.tokens(seed, S)
    q, K, V = G.decode_qkv(seed, S, Hq, Hkv)
    lay = D.build_blocks(t(toks[None]), t(G.T7_IDS), t(K[None], torch.bfloat16), t(V[None], torch.bfloat16),
                         cfg, static_w10=G.T7_W10, Hq=Hq)
    return lay, q, K, V, toks


def test_clean_run_reports_no_error(D):
    lay, q, *_ = _layer(D)
    shape = D.make_shape(1, lay.shape.S, 8, 2)
    ws = torch.zeros(D.workspace_bytes(D.OP_DECODE_LAYER, shape, lay.cfg, 300), dtype=torch.uint8, device=DEV)
    D.decode_layer(t(q[None], torch.bfloat16), lay, 300, ws=ws)
    assert D.read_device_error(ws) == 0


def test_select_plan_coverage(D):
    """A plan whose starts are not strictly increasing: a6 flags
    PlanCoverageMismatch and selects nothing for that sequence."""
    lay, q, *_ = _layer(D)
    bad = lay.block_starts.clone()
    bad[0, 5] = bad[0, 4]                      # an empty block
    lay_bad = D.PagedLayer(**{**lay.__dict__, "block_starts": bad})
    shape = D.make_shape(1, lay.shape.S, 8, 2)
    ws = torch.zeros(D.workspace_bytes(D.OP_SELECT, shape, lay.cfg, 300), dtype=torch.uint8, device=DEV)
    sel = D.select(t(q[None], torch.bfloat16), lay_bad, 300, ws=ws)
    assert D.read_device_error(ws) & D.DEVERR_PLAN_COVERAGE
    assert sel.n_sel.cpu().numpy().tolist() == [[0] * 8]
    cnt = sel.worklist[256:264].view(torch.int32).cpu().numpy()
    assert cnt.tolist() == [0, 0]
    D.clear_device_error(ws)
    assert D.read_device_error(ws) == 0
    # the decode-layer call (fused or three kernels) reports it in its own word
    ws2 = torch.zeros(D.workspace_bytes(D.OP_DECODE_LAYER, shape, lay.cfg, 300), dtype=torch.uint8, device=DEV)
    o, lse, _ = D.decode_layer(t(q[None], torch.bfloat16), lay_bad, 300, ws=ws2)
    assert D.read_device_error(ws2) & D.DEVERR_PLAN_COVERAGE
    assert torch.isneginf(lse).all()            # nothing selected -> lse = -inf


def test_select_plan_end_beyond_capacity(D):
    lay, q, *_ = _layer(D)
    bad = lay.block_starts.clone()
    nb = int(lay.n_blocks[0])
    bad[0, nb] = lay.shape.S + 5                 # last block ends past S
    lay_bad = D.PagedLayer(**{**lay.__dict__, "block_starts": bad})
    shape = D.make_shape(1, lay.shape.S, 8, 2)
    ws = torch.zeros(D.workspace_bytes(D.OP_SELECT, shape, lay.cfg, 300), dtype=torch.uint8, device=DEV)
    D.select(t(q[None], torch.bfloat16), lay_bad, 300, ws=ws)
    assert D.read_device_error(ws) & D.DEVERR_PLAN_COVERAGE


def test_map_pages_coverage_and_capacity(D):
    cfg = D.default_config()
    S = 2000
    toks = G.tokens(5, S)
    bs, nb = D.segment(t(toks[None]), t(G.T7_IDS), t(G.T7_W10[None], torch.uint8), cfg)
    ws = torch.zeros(D.workspace_bytes(D.OP_MAP_PAGES, D.make_shape(1, S, 1, 1), cfg), dtype=torch.uint8,
                     device=DEV)
    pf, pb, pv, npg = D.map_pages(bs, nb, S, cfg, ws=ws)
    assert D.read_device_error(ws) == 0 and int(npg[0]) > 0
    # plan ends before S: not a tiling of [0, S)
    short = bs.clone()
    short[0, int(nb[0])] = S - 3
    _, _, _, npg2 = D.map_pages(short, nb, S, cfg, ws=ws)
    assert D.read_device_error(ws) == D.DEVERR_PLAN_COVERAGE and int(npg2[0]) == -1
    D.clear_device_error(ws)
    # a page capacity smaller than the plan needs
    need = int(npg[0])
    small = D.default_config(page_cap=need - 1)
    _, _, _, npg3 = D.map_pages(bs, nb, S, small, ws=ws)
    assert D.read_device_error(ws) == D.DEVERR_PAGE_CAPACITY and int(npg3[0]) == -1
    D.clear_device_error(ws)
    exact = D.default_config(page_cap=need)
    _, _, _, npg4 = D.map_pages(bs, nb, S, exact, ws=ws)
    assert D.read_device_error(ws) == 0 and int(npg4[0]) == need


def test_repack_skips_bad_plan(D):
    cfg = D.default_config()
    S, Hkv = 1500, 2
    toks = G.tokens(6, S)
    _, K, V = G.decode_qkv(6, S, 4, Hkv)
    bs, nb = D.segment(t(toks[None]), t(G.T7_IDS), t(G.T7_W10[None], torch.uint8), cfg)
    pf, _, _, _ = D.map_pages(bs, nb, S, cfg)
    bad = bs.clone()
    bad[0, 0] = 1                                # does not start at 0
    ws = torch.zeros(256, dtype=torch.uint8, device=DEV)
    D.repack_digest(t(K[None], torch.bfloat16), t(V[None], torch.bfloat16), bad, nb, pf, cfg, ws=ws)
    assert D.read_device_error(ws) & D.DEVERR_PLAN_COVERAGE


def test_select_overflow_clamped(D):
    """A caller-supplied plan with blocks shorter than C - Delta (33 one-token
    blocks, then one long block of zero keys) makes every head select more
    blocks than max_selected: sel_blocks is clamped, the overflow flagged and
    nothing is written past the array."""
    cfg = D.default_config()
    S, Hq, Hkv, budget = 600, 4, 1, 30
    q, K, V = G.decode_qkv(7, S, Hq, Hkv)
    qhat = q.mean(0) / np.linalg.norm(q.mean(0))
    K[:33, 0] = G.to_bf16(5.0 * qhat[None] + 0.05 * K[:33, 0])
    K[33:] = 0.0                                  # the long block scores exactly 0
    mb = D.max_blocks(S, cfg)
    starts = list(range(34)) + [S]                # 34 blocks <= max_blocks
    assert len(starts) - 1 <= mb
    bs = np.full((1, mb + 1), S, np.int32)
    bs[0, : len(starts)] = starts
    bs_d, nb_d = t(bs), t(np.array([len(starts) - 1], np.int32))
    pf, pb, pv, npg = D.map_pages(bs_d, nb_d, S, cfg)
    Kp, Vp, dig = D.repack_digest(t(K[None], torch.bfloat16), t(V[None], torch.bfloat16), bs_d, nb_d, pf, cfg)
    lay = D.PagedLayer(D.make_shape(1, S, Hq, Hkv), cfg, None, bs_d, nb_d, pf, pb, pv, npg, Kp, Vp, dig)
    shape = D.make_shape(1, S, Hq, Hkv)
    ms = D.max_selected(budget, S, cfg)
    ws = torch.zeros(D.workspace_bytes(D.OP_SELECT, shape, cfg, budget), dtype=torch.uint8, device=DEV)
    guard = 4096
    sb_full = torch.full((Hq * ms + guard,), -7, dtype=torch.int32, device=DEV)
    sb = sb_full[: Hq * ms].view(1, Hq, ms)
    _, ns, mg, kp, wl = D._sel_outputs(shape, cfg, budget, DEV, want_blocks=False)
    sel = D.select(t(q[None], torch.bfloat16), lay, budget, out=(sb, ns, mg, kp, wl, None), ws=ws)
    assert D.read_device_error(ws) & D.DEVERR_SELECT_OVERFLOW
    assert int(sel.n_sel.max()) > ms
    assert bool((sb_full[Hq * ms:] == -7).all())   # nothing written past the clamp


def test_append_plan_mismatch(D):
    cfg = D.default_config()
    B, Hq, Hkv, S_cap = 1, 4, 2, 800
    toks = G.tokens(8, S_cap)
    w10 = t(G.T7_W10[None], torch.uint8)
    lay = D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, torch.bfloat16, DEV)
    ws = D.append_workspace(lay)
    _, K, V = G.decode_qkv(8, S_cap, Hq, Hkv)
    Kd, Vd = t(K[None], torch.bfloat16), t(V[None], torch.bfloat16)
    D.append_plan(t(toks[None]), t(G.T7_IDS), lay, 0, 500, ws)
    D.append_kv(lay, Kd[:, :500].contiguous(), Vd[:, :500].contiguous(), 0, 500, ws)
    assert D.read_device_error(ws) == 0
    before = lay.block_starts.clone()
    # the stored plan covers 500 tokens; claiming L_prev = 510 is a PlanMismatch
    D.append_plan(t(toks[None]), t(G.T7_IDS), lay, 510, 511, ws)
    assert D.read_device_error(ws) & D.DEVERR_PLAN_MISMATCH
    assert torch.equal(lay.block_starts, before)     # the sequence was left untouched


def test_append_then_decode_without_sync(D):
    """append_plan + append_kv_layers immediately followed by decode_layer on
    the same stream (no host synchronisation): the PDL prologues of the decode
    kernels must read the appended digests/pages (the fence orders them)."""
    cfg = D.default_config()
    B, Hq, Hkv, S0, n_steps = 1, 8, 2, 2500, 6
    S_cap = S0 + n_steps
    toks = G.tokens(9, S_cap)
    q, K, V = G.decode_qkv(9, S_cap, Hq, Hkv)
    # make the appended tokens decisive: the query attends to them strongly
    K[S0:] = 6.0 * q.reshape(Hkv, Hq // Hkv, -1).mean(1)[None] + 0.1 * K[S0:]
    K = G.to_bf16(K)
    w10 = t(G.T7_W10[None], torch.uint8)
    lay = D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, torch.bfloat16, DEV)
    ws = D.append_workspace(lay)
    Kd, Vd = t(K[None], torch.bfloat16), t(V[None], torch.bfloat16)
    ids, td = t(G.T7_IDS), t(toks[None])
    D.append_plan(td, ids, lay, 0, S0, ws)
    D.append_kv(lay, Kd[:, :S0].contiguous(), Vd[:, :S0].contiguous(), 0, S0, ws)
    budget = 200
    qt = t(q[None], torch.bfloat16)
    outs = []
    L = S0
    for i in range(n_steps):
        D.append_plan(td, ids, lay, L, L + 1, ws)
        D.append_kv(lay, Kd[:, L:L + 1].contiguous(), Vd[:, L:L + 1].contiguous(), L, L + 1, ws)
        L += 1
        o, lse, sel = D.decode_layer(qt, lay, budget)      # no synchronize in between
        outs.append((L, o.clone(), lse.clone()))
    torch.cuda.synchronize()
    for L, o, lse in outs:
        st = O.segment(toks[:L], G.T7_IDS, G.T7_W10, cfg.C, cfg.delta)
        res = O.decode_step(q, K[:L], V[:L], st, budget)
        err = H.row_rel_err(o[0].cpu().numpy(), res["o"])
        assert np.all(err <= 2e-3), (L, err.max())
        assert np.allclose(lse[0].cpu().numpy(), res["lse"], atol=1e-4, rtol=1e-4)


def test_attention_nw4_g8_subprocess():
    """DYNSPLIT_ATTN_NW=4 with G = 8 (more heads than warps): every head's
    output must be written by the split merge."""
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, %r)
from paper_2602_03184_b200 import dynsplit as D
from oracle import dynsplit_oracle as O
from synth import generators as G
from tests import helpers as H
S, Hq, Hkv, budget = 6000, 16, 2, 1500
toks = G.tokens(31, S)
q, K, V = G.decode_qkv(31, S, Hq, Hkv)
st = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
q = H.certify_queries(31, q[None], K[None], [st], budget)[0]
t = lambda x, dt=None: torch.as_tensor(np.ascontiguousarray(x)).to("cuda:0", dtype=dt)
cfg = D.default_config()
lay = D.build_blocks(t(toks[None]), t(G.T7_IDS), t(K[None], torch.bfloat16), t(V[None], torch.bfloat16), cfg,
                     static_w10=G.T7_W10, Hq=Hq)
qt = t(q[None], torch.bfloat16)
sel = D.select(qt, lay, budget)
o, lse = D.decode_attn(qt, lay, sel.worklist)
torch.cuda.synchronize()
res = O.decode_step(q, K, V, st, budget)
err = H.row_rel_err(o[0].cpu().numpy(), res["o"])
assert np.all(err <= 2e-3), err
assert np.allclose(lse[0].cpu().numpy(), res["lse"], atol=1e-4, rtol=1e-4)
print("ok")
''' % ROOT
    env = dict(os.environ, DYNSPLIT_ATTN_NW="4")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_append_kv_without_plan_append(D):
    """append_kv for [L, L + 1) without the matching append_plan: the
    workspace still describes the previous append, so the kernel reports a
    PlanMismatch and writes nothing (the staged tail would not match)."""
    cfg = D.default_config()
    B, Hq, Hkv, S_cap = 1, 4, 2, 800
    toks = G.tokens(8, S_cap)
    w10 = t(G.T7_W10[None], torch.uint8)
    lay = D.alloc_paged(B, S_cap, Hq, Hkv, cfg, w10, torch.bfloat16, DEV)
    ws = D.append_workspace(lay)
    _, K, V = G.decode_qkv(8, S_cap, Hq, Hkv)
    Kd, Vd = t(K[None], torch.bfloat16), t(V[None], torch.bfloat16)
    D.append_plan(t(toks[None]), t(G.T7_IDS), lay, 0, 500, ws)
    D.append_kv(lay, Kd[:, :500].contiguous(), Vd[:, :500].contiguous(), 0, 500, ws)
    assert D.read_device_error(ws) == 0
    kp, vp, dg = lay.Kp.clone(), lay.Vp.clone(), lay.digests.clone()
    D.append_kv(lay, Kd[:, 500:501].contiguous(), Vd[:, 500:501].contiguous(), 500, 501, ws)
    assert D.read_device_error(ws) & D.DEVERR_PLAN_MISMATCH
    assert torch.equal(lay.Kp, kp) and torch.equal(lay.Vp, vp) and torch.equal(lay.digests, dg)


def test_fused_synccheck_subprocess():
    """compute-sanitizer synccheck + memcheck over the decode-model flow
    (append kernels, then the fused layer reusing their shared memory): every
    mbarrier is initialised before any thread polls it (a stale word once read
    as a completed phase) and no access is out of bounds."""
    import shutil
    san = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(san):
        pytest.skip("compute-sanitizer not available")
    for tool in ("synccheck", "memcheck"):
        r = subprocess.run([san, "--tool", tool, "--error-exitcode", "9", sys.executable,
                            os.path.join(ROOT, "tests", "_san_append_decode.py")],
                           capture_output=True, text=True, timeout=600, cwd=ROOT)
        if r.returncode != 0 and "closed" in r.stderr and not r.stdout:
            pytest.skip("compute-sanitizer is closed on this GPU pool: " + r.stderr.strip()[:120])
        assert r.returncode == 0 and "ok" in r.stdout, (tool, r.stdout[-3000:], r.stderr[-3000:])

"""NEXT-4: end-to-end decoding through random-weight Llama-shaped layers
(paper_2602_03184_b200/model.py) on a reduced shape.

* the device-position append keeps the shared plan equal to the oracle's
  DD-Select of the whole token stream after every generated token;
* the sparse model with a budget covering the context equals the dense model
  (our dense a9 kernel) step by step;
* both agree with an independent plain-torch model (fp32 softmax attention
  over a token-major cache built from the same projections) within bf16
  tolerance;
* one decode step captured as a CUDA graph and replayed gives the same tokens
  and logits as eager steps.
"""
import numpy as np
import pytest
import torch

from oracle import dynsplit_oracle as O
from synth import generators as G

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _model(attn, budget, B=2, S0=600, S_cap=700, seed=5):
    from paper_2602_03184_b200 import dynsplit as D
    from paper_2602_03184_b200.model import LlamaShape, RandomLlama
    sh = LlamaShape(layers=2, d_model=256, Hq=4, Hkv=2, d=128, ffn=512, vocab=32000)  # the synthetic ids < 32000
    ids = torch.from_numpy(G.T7_IDS).to(DEV)
    w10 = torch.from_numpy(np.tile(G.T7_W10, (B, 1))).to(torch.uint8)
    m = RandomLlama(sh, B, S_cap, budget, DEV, seed=seed, attn=attn, delim_ids=ids, w10=w10)
    toks = torch.from_numpy(np.stack([G.tokens(4000 + b, S0) for b in range(B)])).to(DEV)
    m.prefill_synthetic(toks, seed=seed + 1)
    return m


def _stream(B, n, S0=600):
    """Teacher-forced continuation tokens (delimiter-rich, as the prompt)."""
    return torch.from_numpy(np.stack([G.tokens(4100 + b, S0 + n)[S0:] for b in range(B)])).to(DEV)


def test_plan_follows_oracle_while_generating():
    B, n = 2, 60
    m = _model("sparse", 64)
    cont = _stream(B, n)
    for i in range(n):
        m.step(cont[:, i].contiguous())
    torch.cuda.synchronize()
    L = 600 + n
    assert int(m.pos.item()) == L
    toks = m.tokens[:, :L].cpu().numpy()
    for b in range(B):
        starts = O.segment(toks[b], G.T7_IDS, G.T7_W10, 32, 14)
        nb = int(m.layers[0].n_blocks[b])
        assert m.layers[0].block_starts[b, : nb + 1].tolist() == starts
    from paper_2602_03184_b200 import dynsplit as D
    assert D.read_device_error(m.ws_app) == 0


def test_sparse_full_budget_equals_dense_model():
    """Budget >= the context: every block is selected, so the sparse model's
    attention must match the dense model's (a different kernel path) at every
    layer and step; tokens are teacher-forced."""
    B, n = 2, 12
    ms, md = _model("sparse", 10 ** 6), _model("dense", 10 ** 6)
    cont = _stream(B, n)
    worst = 0.0
    for i in range(n):
        ts = ms.step(cont[:, i].contiguous())
        td = md.step(cont[:, i].contiguous())
        os_, od = ms.o.float(), md.o.float()
        err = ((os_ - od).abs().amax(-1) / od.abs().amax(-1).clamp_min(1e-6)).max().item()
        worst = max(worst, err)
        assert torch.allclose(ms.lse, md.lse, rtol=0, atol=1e-3)
    assert worst <= 2e-3, worst


def test_against_plain_torch_model():
    """An independent plain-torch decoder (the model's weights, a token-major
    KV cache with the prompt's K/V read back from the pages, fp32 softmax
    attention over every token) gives the same next tokens and close final
    hidden states when the sparse model's budget covers the context."""
    from paper_2602_03184_b200 import dynsplit as D
    B, n, S0 = 2, 8, 600
    m = _model("sparse", 10 ** 6)
    sh = m.sh
    # the prompt's K/V back from the pages (oracle unpack of the plan)
    starts = [O.segment(m.tokens[b, :S0].cpu().numpy(), G.T7_IDS, G.T7_W10, 32, 14) for b in range(B)]
    Kc, Vc = [], []
    for l in range(sh.layers):
        lay = m.layers[l]
        Kc.append([torch.from_numpy(O.unpack(lay.Kp[b].float().cpu().numpy(), starts[b], 16)).float().to(DEV)
                   for b in range(B)])
        Vc.append([torch.from_numpy(O.unpack(lay.Vp[b].float().cpu().numpy(), starts[b], 16)).float().to(DEV)
                   for b in range(B)])
    cont = _stream(B, n)
    pos = S0
    nq, nk = sh.Hq * sh.d, sh.Hkv * sh.d
    g = sh.Hq // sh.Hkv
    for i in range(n):
        tok = cont[:, i].contiguous()
        t_ours = m.step(tok)
        # reference step
        x = m.emb.index_select(0, tok.long())
        cos, sin = m.cos[pos][None, None, :], m.sin[pos][None, None, :]
        for l in range(sh.layers):
            h = torch.nn.functional.rms_norm(x, (sh.d_model,), m.n1[l], sh.eps)
            qkv = h @ m.w_qkv[l]
            q = m._rope(qkv[:, :nq].float().view(B, sh.Hq, sh.d), cos, sin).to(torch.bfloat16)
            k = m._rope(qkv[:, nq:nq + nk].float().view(B, sh.Hkv, sh.d), cos, sin).to(torch.bfloat16)
            v = qkv[:, nq + nk:].reshape(B, sh.Hkv, sh.d)
            outs = []
            for b in range(B):
                Kc[l][b] = torch.cat([Kc[l][b], k[b][None].float()])
                Vc[l][b] = torch.cat([Vc[l][b], v[b][None].float()])
                Kb = Kc[l][b].repeat_interleave(g, dim=1)          # [T, Hq, d]
                Vb = Vc[l][b].repeat_interleave(g, dim=1)
                z = torch.einsum("hd,thd->ht", q[b].float(), Kb) / sh.d ** 0.5
                outs.append(torch.einsum("ht,thd->hd", torch.softmax(z, -1), Vb))
            o = torch.stack(outs)
            x = x + o.view(B, nq).to(torch.bfloat16) @ m.w_o[l]
            h2 = torch.nn.functional.rms_norm(x, (sh.d_model,), m.n2[l], sh.eps)
            gu = h2 @ m.w_gu[l]
            x = x + (torch.nn.functional.silu(gu[:, :sh.ffn]) * gu[:, sh.ffn:]) @ m.w_down[l]
        logits = torch.nn.functional.rms_norm(x, (sh.d_model,), m.nf, sh.eps) @ m.emb.t()
        t_ref = logits.argmax(-1).to(torch.int32)
        top2 = logits.float().topk(2, dim=-1).values
        decided = (top2[:, 0] - top2[:, 1]) > 1e-2 * top2[:, 0].abs().clamp_min(1.0)
        assert torch.equal(t_ours[decided], t_ref[decided])
        pos += 1


def test_graph_replay_equals_eager():
    """The device-resident decode step (append with the position in device
    memory, fused attention, cuBLAS projections, argmax) captured once and
    replayed per token equals eager steps bit for bit."""
    B, n = 2, 6
    me, mg = _model("sparse", 300), _model("sparse", 300)
    cont = _stream(B, n)
    eager = [me.step(cont[:, i].contiguous()).clone() for i in range(n)]
    tok_in = cont[:, 0].contiguous().clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        out0 = mg.step(tok_in)          # eager step 0 (also sets the kernel attributes)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    assert torch.equal(out0, eager[0])
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = mg.step(tok_in)           # recorded, not run
    for i in range(1, n):
        tok_in.copy_(cont[:, i])
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager[i]), i
    assert torch.equal(mg.o, me.o) and int(mg.pos.item()) == int(me.pos.item())

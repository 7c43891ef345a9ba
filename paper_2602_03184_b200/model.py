"""NEXT-4: end-to-end decoding through random-weight Llama-shaped layers
(the shape of the paper's Fig. 8: sparse vs dense
decode latency over generated lengths at a long input).

The model is plumbing around the hot path: embeddings, RMSNorm, the QKV / O /
gated-MLP projections (plain cuBLAS GEMMs through torch.matmul, as the task
allows for plain library GEMMs), RoPE and the argmax sampler are torch ops;
every step of the DynSplit-KV path runs in libdynsplit kernels:
  * the new token is appended to the shared DD-Select plan and to every
    layer's pages and digests (dynsplit_append_plan_dev /
    dynsplit_append_kv_layers_dev: NEXT-1, incremental re-segmentation of the
    tail);
  * attention is dynsplit_decode_layer (the fused a5-a8 kernel) -- or, for the
    baseline, dynsplit_decode_attn in dense mode (a9) over every page.
The decode position lives in device memory, so one decode step (all layers)
is captured once as a CUDA graph and replayed per generated token.

Weights are random (no checkpoints are available): W ~ N(0, 1/fan_in), bf16.
Nothing here claims accuracy; it measures what a decode step costs.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import torch

from . import dynsplit as D


@dataclass
class LlamaShape:
    """Llama-3-8B by default (32 layers, 4096 model dim, 32 Q / 8 KV heads of
    128, SwiGLU 14336, vocabulary 128256, RoPE theta 5e5)."""
    layers: int = 32
    d_model: int = 4096
    Hq: int = 32
    Hkv: int = 8
    d: int = 128
    ffn: int = 14336
    vocab: int = 128256
    rope_theta: float = 500000.0
    eps: float = 1e-5


class RandomLlama:
    """Random-weight Llama-shaped decoder over a DynSplit-KV paged cache for B
    sequences of capacity S_cap tokens.  attn = "sparse" (budgeted selection,
    dynsplit_decode_layer) or "dense" (every page, dynsplit_decode_attn)."""

    def __init__(self, shape: LlamaShape, B: int, S_cap: int, budget: int, device, seed: int = 0,
                 attn: str = "sparse", cfg: Optional[D.Config] = None, delim_ids=None, w10=None):
        assert attn in ("sparse", "dense")
        self.sh, self.B, self.S_cap, self.budget, self.attn = shape, B, S_cap, budget, attn
        dev = torch.device(device)
        self.dev = dev
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        bf = torch.bfloat16
        sh = shape

        def w(rows, cols):
            return (torch.randn(rows, cols, generator=g, device=dev) / rows ** 0.5).to(bf)

        self.emb = (torch.randn(sh.vocab, sh.d_model, generator=g, device=dev) * 0.02).to(bf)  # tied LM head
        nq, nk = sh.Hq * sh.d, sh.Hkv * sh.d
        self.w_qkv = [w(sh.d_model, nq + 2 * nk) for _ in range(sh.layers)]
        self.w_o = [w(nq, sh.d_model) for _ in range(sh.layers)]
        self.w_gu = [w(sh.d_model, 2 * sh.ffn) for _ in range(sh.layers)]
        self.w_down = [w(sh.ffn, sh.d_model) for _ in range(sh.layers)]
        self.n1 = [torch.ones(sh.d_model, device=dev, dtype=bf) for _ in range(sh.layers)]
        self.n2 = [torch.ones(sh.d_model, device=dev, dtype=bf) for _ in range(sh.layers)]
        self.nf = torch.ones(sh.d_model, device=dev, dtype=bf)
        # RoPE tables [S_cap, d / 2]
        inv = 1.0 / (sh.rope_theta ** (torch.arange(0, sh.d, 2, device=dev, dtype=torch.float32) / sh.d))
        ang = torch.arange(S_cap, device=dev, dtype=torch.float32)[:, None] * inv[None]
        self.cos, self.sin = ang.cos(), ang.sin()
        self.cos2 = torch.cat([self.cos, self.cos], -1)  # [S_cap, d] for the fused rotate-half form
        self.sin2 = torch.cat([self.sin, self.sin], -1)
        # the paged cache: one plan shared by every layer
        self.cfg = cfg if cfg is not None else D.default_config()
        self.delim_ids = delim_ids
        w10 = w10.to(dev) if w10 is not None else None
        self.layers: List[D.PagedLayer] = []
        for l in range(sh.layers):
            self.layers.append(D.alloc_paged(B, S_cap, sh.Hq, sh.Hkv, self.cfg, w10, device=dev,
                                             plan_from=self.layers[0] if l else None))
        self.tokens = torch.zeros(B, S_cap, dtype=torch.int32, device=dev)
        self.pos = torch.zeros(1, dtype=torch.int32, device=dev)        # tokens already in the cache
        self.ws_app = D.append_workspace(self.layers[0])
        dshape = D.make_shape(B, S_cap, sh.Hq, sh.Hkv, sh.d)
        self.dshape = dshape
        self.ws_dec = D.workspace(D.workspace_bytes(D.OP_DECODE_LAYER, dshape, self.cfg, budget), dev, "model_dec")
        _, self.ns, self.mg, self.kp, self.wl = D._sel_outputs(dshape, self.cfg, budget, dev, want_blocks=False)
        self.o = torch.empty(B, sh.Hq, sh.d, device=dev)
        self.lse = torch.empty(B, sh.Hq, device=dev)

    # ------------------------------------------------------------------ cache
    def prefill_synthetic(self, tokens: torch.Tensor, seed: int = 1, k_scale: float = 1.5):
        """Fill the cache with a synthetic prompt: tokens [B, S0] (int32,
        device) and random K/V per layer (the bench's distribution), planned
        and paged through the append path from an empty cache (L_prev = 0)."""
        B, S0 = tokens.shape
        sh = self.sh
        self.tokens[:, :S0] = tokens
        lay0 = self.layers[0]
        D.append_plan(self.tokens, self.delim_ids, lay0, 0, S0, self.ws_app)
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        for l in range(sh.layers):
            K = (k_scale * torch.randn(B, S0, sh.Hkv, sh.d, generator=g, device=self.dev)).to(torch.bfloat16)
            V = torch.randn(B, S0, sh.Hkv, sh.d, generator=g, device=self.dev).to(torch.bfloat16)
            D.append_kv(self.layers[l], K, V, 0, S0, self.ws_app)
            del K, V
        self.pos.fill_(S0)

    # ------------------------------------------------------------------ decode
    def _rope(self, x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
        """Rotate [B, H, d] (fp32) by the position's angles (rotate-half form)."""
        h = x.shape[-1] // 2
        x1, x2 = x[..., :h], x[..., h:]
        return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)

    def step(self, tok: torch.Tensor) -> torch.Tensor:
        """One decode step for the B sequences: tok int32 [B] (device) is the
        token at position pos; returns the next tokens (argmax, int32 [B]).
        Everything stays on the device (graph-capturable)."""
        sh, B = self.sh, self.B
        nq, nk = sh.Hq * sh.d, sh.Hkv * sh.d
        # the token joins the sequence; the shared plan grows by one (NEXT-1)
        self.tokens.scatter_(1, self.pos.long().expand(B, 1), tok[:, None])
        D.append_plan_dev(self.tokens, self.delim_ids, self.layers[0], self.pos, 1, self.ws_app)
        cos2 = self.cos2.index_select(0, self.pos.long())[:, None, :]               # [1, 1, d]
        sin2 = self.sin2.index_select(0, self.pos.long())[:, None, :]
        hd = sh.d // 2
        x = self.emb.index_select(0, tok.long())                                   # [B, dm] bf16
        for l in range(sh.layers):
            h = torch.nn.functional.rms_norm(x, (sh.d_model,), self.n1[l], sh.eps)
            qkv = h @ self.w_qkv[l]
            # RoPE of q and k together (rotate-half form, fp32): x cos + [-x2 | x1] sin
            qk = qkv[:, :nq + nk].float().view(B, sh.Hq + sh.Hkv, sh.d)
            qk = torch.addcmul(qk * cos2, torch.cat([-qk[..., hd:], qk[..., :hd]], -1), sin2).to(torch.bfloat16)
            q = qk[:, :sh.Hq].contiguous()
            k = qk[:, sh.Hq:].unsqueeze(1).contiguous()                            # [B, 1, Hkv, d]
            v = qkv[:, nq + nk:].view(B, 1, sh.Hkv, sh.d).contiguous()
            D.append_kv_layers_dev([self.layers[l]], [k], [v], self.pos, 1, self.ws_app)
            if self.attn == "sparse":
                D.decode_layer(q, self.layers[l], self.budget,
                               out=(self.ns, self.mg, self.kp, self.wl, self.o, self.lse), ws=self.ws_dec)
            else:
                D.decode_attn(q, self.layers[l], None, out=(self.o, self.lse), ws=self.ws_dec)
            x = torch.addmm(x, self.o.view(B, nq).to(torch.bfloat16), self.w_o[l])  # residual add in the GEMM
            h2 = torch.nn.functional.rms_norm(x, (sh.d_model,), self.n2[l], sh.eps)
            gu = h2 @ self.w_gu[l]
            x = torch.addmm(x, torch.nn.functional.silu(gu[:, :sh.ffn]).mul_(gu[:, sh.ffn:]), self.w_down[l])
        logits = torch.nn.functional.rms_norm(x, (sh.d_model,), self.nf, sh.eps) @ self.emb.t()
        self.pos.add_(1)
        return logits.argmax(dim=-1).to(torch.int32)


def time_decode(model: RandomLlama, first_tok: torch.Tensor, checkpoints, warmup: int = 3):
    """Generate tokens with one decode step captured as a CUDA graph (the
    step's argmax feeds the next replay on the device) and return, for every
    checkpoint n in `checkpoints` (ascending), the mean ms per token of the
    tokens generated up to n (CUDA events).  The first `warmup` steps run
    eagerly (kernel attributes, cuBLAS heuristics) and count as generated."""
    dev = first_tok.device
    tok = first_tok.clone()
    for _ in range(warmup):
        tok = model.step(tok)
    tok_in = tok.clone()
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = model.step(tok_in)
        tok_in.copy_(out)
    cur = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(checkpoints) + 1)]
    ev[0].record(cur)
    done = warmup
    res = {}
    for i, n in enumerate(checkpoints):
        while done < n:
            g.replay()
            done += 1
        ev[i + 1].record(cur)
    torch.cuda.synchronize()
    prev = warmup
    tot = 0.0
    for i, n in enumerate(checkpoints):
        tot += ev[i].elapsed_time(ev[i + 1])
        res[n] = tot / max(n - warmup, 1)
    del g
    return res

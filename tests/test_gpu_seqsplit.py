"""Sequence split (BASELINE config 4) through the kernels on one GPU.

* test_seq_split_two_processes: `parallel.SeqSplitDecoder.step` itself -- a5
  into the send buffer, the real all-gathers (gloo, both ranks on cuda:0: the
  one-GPU lease has no second device for NCCL), the index gather, a6 with the
  rank's block range, a7, the partial all-gathers and the rank-ordered a8
  merge -- against the oracle; both ranks must produce identical merged
  outputs and selections equal to the single-GPU call.
* test_seq_split_emulated: the same buffers and index map with the
  all-gather replaced by concatenating the ranks' send buffers (what the
  collective does), for several world sizes in one process.
"""
import os
import socket
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


def t(x, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(x)).to(DEV, dtype=dtype)


def _problem(Hq, Hkv, S, budget, seed=1400):
    toks = G.tokens(seed, S)
    q, K, V = G.decode_qkv(seed + 1, S, Hq, Hkv)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
    q = H.certify_queries(seed + 1, q[None], K[None], [starts], budget)[0]
    return toks, q, K, V, starts


@pytest.mark.parametrize("world,Hq,Hkv,S,budget", [(2, 32, 8, 8192, 1024), (4, 8, 8, 6000, 700),
                                                   (3, 16, 2, 5000, 16), (8, 40, 40, 9000, 1200)])
def test_seq_split_emulated(world, Hq, Hkv, S, budget):
    from paper_2602_03184_b200 import dynsplit as D
    from paper_2602_03184_b200 import parallel as PAR
    cfg = D.default_config()
    toks, q, K, V, starts = _problem(Hq, Hkv, S, budget)
    glob, ranges = PAR.global_plan(t(toks[None]), t(G.T7_IDS), cfg, G.T7_W10, Hq, Hkv, world)
    assert glob.block_starts[0, : int(glob.n_blocks[0]) + 1].tolist() == starts
    qt = t(q[None], torch.bfloat16)
    decs, lays = [], []
    for r in range(world):
        t_lo, t_hi = PAR.shard_token_range(starts, ranges, r)
        lays.append(PAR.local_layer(glob, ranges, r, t(K[None, t_lo:t_hi], torch.bfloat16),
                                    t(V[None, t_lo:t_hi], torch.bfloat16), cfg, Hq))
        decs.append(PAR.SeqSplitDecoder(glob, ranges, r, Hq, budget, DEV))
    # a5 per rank into its send buffer; the all-gather = concatenation
    for dec, lay in zip(decs, lays):
        D.score_blocks(qt, lay, out=dec.send[: Hq * dec.stride].view(1, Hq, dec.stride))
    cat = torch.cat([dec.send for dec in decs])
    parts_o, parts_l = [], []
    for dec, lay in zip(decs, lays):
        dec.gathered[: cat.numel()].copy_(cat)
        torch.index_select(dec.gathered, 0, dec.idx, out=dec.scores.view(-1))
        sel = D.select_from_scores(dec.scores, glob, budget, Hq, blk_lo=dec.lo, blk_hi=dec.hi, out=dec.sel_out,
                                   ws=dec.ws_sel)
        o, l = D.decode_attn(qt, lay, sel.worklist)
        parts_o.append(o.reshape(Hq, -1))
        parts_l.append(l.reshape(Hq))
    o, lse = D.merge_partials(torch.stack(parts_o).contiguous(), torch.stack(parts_l).contiguous())
    torch.cuda.synchronize()
    ref = O.decode_step(q, K, V, starts, budget)
    err = H.row_rel_err(o.cpu().numpy(), ref["o"])
    assert np.all(err <= 2e-3), err.max()
    assert np.all(np.abs(lse.cpu().numpy() - ref["lse"]) <= 1e-4 * np.maximum(1, np.abs(ref["lse"])))
    # every rank's global scores and selection equal one single-GPU scoring of the whole sequence
    single = D.build_blocks(t(toks[None]), t(G.T7_IDS), t(K[None], torch.bfloat16), t(V[None], torch.bfloat16),
                            cfg, static_w10=G.T7_W10, Hq=Hq)
    sel1 = D.select(qt, single, budget)
    nb = len(starts) - 1
    for dec in decs:
        assert torch.equal(dec.scores[..., :nb], sel1.scores[..., :nb])
        ns, mg, kp = dec.selection()
        assert torch.equal(ns, sel1.n_sel) and torch.equal(mg, sel1.marginal_block)
        assert torch.equal(kp, sel1.marginal_keep)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_WORKER = r'''
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ROOT)
from paper_2602_03184_b200 import dynsplit as D
from paper_2602_03184_b200 import parallel as PAR
from oracle import dynsplit_oracle as O
from synth import generators as G
from tests import helpers as H
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
Hq, Hkv, S, budget, L = 32, 8, 9000, 1024, 3
t = lambda x, dt=None: torch.as_tensor(np.ascontiguousarray(x)).to("cuda:0", dtype=dt)
cfg = D.default_config()
toks = G.tokens(1700, S)
starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
glob, ranges = PAR.global_plan(t(toks[None]), t(G.T7_IDS), cfg, G.T7_W10, Hq, Hkv, world)
dec = PAR.SeqSplitDecoder(glob, ranges, rank, Hq, budget, "cuda:0")
t_lo, t_hi = PAR.shard_token_range(starts, ranges, rank)
ok = True
for l in range(L):                      # several layers through one decoder
    q, K, V = G.decode_qkv(1701 + l, S, Hq, Hkv)
    q = H.certify_queries(1701 + l, q[None], K[None], [starts], budget)[0]
    lay = PAR.local_layer(glob, ranges, rank, t(K[None, t_lo:t_hi], torch.bfloat16),
                          t(V[None, t_lo:t_hi], torch.bfloat16), cfg, Hq)
    o, lse = dec.step(t(q[None], torch.bfloat16), lay)
    torch.cuda.synchronize()
    ref = O.decode_step(q, K, V, starts, budget)
    err = H.row_rel_err(o.cpu().numpy(), ref["o"])
    ok &= bool(np.all(err <= 2e-3))
    ok &= bool(np.all(np.abs(lse.cpu().numpy() - ref["lse"]) <= 1e-4 * np.maximum(1, np.abs(ref["lse"]))))
    ns = dec.selection()[0].cpu().numpy()[0]
    ok &= [len(s) for s in ref["sel_blocks"]] == ns.tolist()
    # both ranks hold bit-identical merged outputs
    both = [torch.empty_like(o).cpu() for _ in range(world)]
    dist.all_gather(both, o.cpu())
    ok &= all(torch.equal(both[0], b) for b in both)
print("RESULT", rank, ok, flush=True)
dist.destroy_process_group()
'''


def test_seq_split_two_processes():
    import subprocess
    port = _free_port()
    code = "ROOT = %r\n" % ROOT + _WORKER
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   LOCAL_RANK="0")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env, cwd=ROOT, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=900) for p in procs]
    for p, (so, se) in zip(procs, outs):
        assert p.returncode == 0, se[-3000:]
        assert "RESULT" in so and so.strip().split()[-1] == "True", so + se[-2000:]

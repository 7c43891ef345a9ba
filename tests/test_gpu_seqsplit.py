"""Sequence split (BASELINE config 4) through the kernels on one GPU: the
ranks are emulated one after another with the same plumbing as the NCCL path
(parallel.assemble_global_scores is what gather_block_scores runs after the
all-gather; dynsplit_merge_partials merges in rank order).  The merged result
must equal the oracle, and every rank's global selection must equal the
single-GPU selection bit-for-bit."""
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


@pytest.mark.parametrize("world,Hq,Hkv,S,budget", [(2, 32, 8, 8192, 1024), (4, 8, 8, 6000, 700),
                                                   (3, 16, 2, 5000, 16)])
def test_seq_split_emulated(world, Hq, Hkv, S, budget):
    from paper_2602_03184_b200 import dynsplit as D
    from paper_2602_03184_b200 import parallel as PAR
    d = 128
    cfg = D.default_config()
    toks = G.tokens(1400, S)
    q, K, V = G.decode_qkv(1401, S, Hq, Hkv, d)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
    q = H.certify_queries(1401, q[None], K[None], [starts], budget)[0]
    glob, ranges = PAR.global_plan(t(toks[None]), t(G.T7_IDS), cfg, G.T7_W10, Hq, Hkv, world)
    assert glob.block_starts[0, : int(glob.n_blocks[0]) + 1].tolist() == starts
    qt = t(q[None], torch.bfloat16)
    shards, bufs = [], []
    for r in range(world):
        t_lo, t_hi = PAR.shard_token_range(starts, ranges, r)
        sh = PAR.build_seq_shard(glob, ranges, r, t(K[None, t_lo:t_hi], torch.bfloat16),
                                 t(V[None, t_lo:t_hi], torch.bfloat16), cfg, Hq)
        shards.append(sh)
        bufs.append(PAR.shard_scores(qt, sh))
    nb = len(starts) - 1
    pad = max(hi - lo for lo, hi in ranges)
    bufs = [torch.nn.functional.pad(b_[..., :pad], (0, max(0, pad - b_.shape[-1])), value=float("-inf"))
            for b_ in bufs]
    gscores = PAR.assemble_global_scores(bufs, ranges, nb)
    outs = [PAR.shard_attend(qt, sh, gscores, budget) for sh in shards]
    o_all = torch.stack([o[0].reshape(Hq, d) for o in outs])
    l_all = torch.stack([o[1].reshape(Hq) for o in outs])
    o, lse = D.merge_partials(o_all.contiguous(), l_all.contiguous())
    torch.cuda.synchronize()
    ref = O.decode_step(q, K, V, starts, budget)
    err = H.row_rel_err(o.cpu().numpy(), ref["o"])
    assert np.all(err <= 2e-3), err.max()
    assert np.all(np.abs(lse.cpu().numpy() - ref["lse"]) <= 1e-4 * np.maximum(1, np.abs(ref["lse"])))
    # the block scores computed on the shards equal a single-GPU scoring of the whole sequence
    single = D.build_blocks(t(toks[None]), t(G.T7_IDS), t(K[None], torch.bfloat16),
                            t(V[None], torch.bfloat16), cfg, static_w10=G.T7_W10, Hq=Hq)
    sel1 = D.select(qt, single, budget)
    assert torch.equal(gscores[..., :nb], sel1.scores[..., :nb])
    for _, _, sel in outs:
        assert torch.equal(sel.n_sel, sel1.n_sel)
        assert torch.equal(sel.marginal_block, sel1.marginal_block)
        assert torch.equal(sel.marginal_keep, sel1.marginal_keep)

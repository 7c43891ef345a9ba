"""Multi-GPU plumbing for the DynSplit-KV hot path (torch.distributed).

Two partitions:

* Batch / KV-group partition (BASELINE config 3): each rank owns whole
  sequences, runs the single-GPU path on them, and nothing crosses the
  interconnect on the data path.  `batch_shard` gives a rank's sequences.

* Sequence split (config 4): every rank holds the global DD-Select plan
  (block boundaries are a cheap function of the tokens) and the pages and
  digests of a contiguous range of blocks.  Per decode step and layer:
    1. local block scores (a5) on the local digests;
    2. all-gather of the scores -> every rank assembles the identical global
       score vector (exact copies), so the budgeted top-k (a6) is global and
       bit-identical on all ranks; the worklist keeps only local pages;
    3. local split-K attention (a7) -> (o_r, lse_r); a rank with nothing
       selected for a head yields lse = -inf, o = 0;
    4. all-gather of (o_r, lse_r) and the log-sum-exp merge (a8) in rank
       order (`dynsplit_merge_partials`).

All compute runs in libdynsplit kernels; this module only moves tensors and
slices plans.  The collective helpers take plain tensors so they are tested
with the gloo backend on CPU (tests/test_parallel_gloo.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist


def batch_shard(n_items: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of n_items for `rank`."""
    base, rem = divmod(n_items, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def seq_split_ranges(block_starts: Sequence[int], n_blocks: int, world: int) -> List[Tuple[int, int]]:
    """Cut the blocks of one sequence into `world` contiguous ranges at the
    block boundary nearest r*S/world (r = 1..world-1); ranges may be empty."""
    bs = [int(x) for x in block_starts[: n_blocks + 1]]
    S = bs[-1]
    cuts = [0]
    j = 0
    for r in range(1, world):
        target = r * S / world
        while j < n_blocks and abs(bs[j + 1] - target) <= abs(bs[j] - target):
            j += 1
        cuts.append(max(j, cuts[-1]))
    cuts.append(n_blocks)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def local_plan(block_starts: torch.Tensor, lo: int, hi: int, max_blocks_local: int):
    """The global plan restricted to blocks [lo, hi), shifted to start at
    token 0 and padded like dynsplit_segment's output (padding = S_local)."""
    seg = block_starts[lo: hi + 1].to(torch.int64)
    base = int(seg[0]) if seg.numel() else 0
    s_local = int(seg[-1]) - base if seg.numel() else 0
    out = torch.full((max_blocks_local + 1,), s_local, dtype=torch.int32, device=block_starts.device)
    out[: hi - lo + 1] = (seg - base).to(torch.int32)
    return out, base, s_local


def gather_block_scores(local_scores: torch.Tensor, ranges: Sequence[Tuple[int, int]],
                        n_global: int, group=None) -> torch.Tensor:
    """All-gather local block scores [..., n_local_pad] (valid prefix = the
    rank's range length) into the global [..., n_global] array; padding is
    -inf.  Every rank ends with bit-identical global scores."""
    world = dist.get_world_size(group)
    pad = max(hi - lo for lo, hi in ranges)
    lead = local_scores.shape[:-1]
    mine = torch.full((*lead, max(pad, 1)), float("-inf"), dtype=local_scores.dtype,
                      device=local_scores.device)
    r = dist.get_rank(group)
    n_mine = ranges[r][1] - ranges[r][0]
    mine[..., :n_mine] = local_scores[..., :n_mine]
    bufs = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(bufs, mine.contiguous(), group=group)
    return assemble_global_scores(bufs, ranges, n_global)


def assemble_global_scores(bufs, ranges, n_global: int) -> torch.Tensor:
    """Place each rank's (padded) local scores at its global block range."""
    lead = bufs[0].shape[:-1]
    out = torch.full((*lead, n_global), float("-inf"), dtype=bufs[0].dtype, device=bufs[0].device)
    for rr, (lo, hi) in enumerate(ranges):
        out[..., lo:hi] = bufs[rr][..., : hi - lo]
    return out


def gather_partials(o: torch.Tensor, lse: torch.Tensor, group=None):
    """All-gather per-rank attention partials -> ([world, rows, d], [world, rows]) in rank order."""
    world = dist.get_world_size(group)
    rows = lse.numel()
    d = o.shape[-1]
    ob = [torch.empty(rows, d, dtype=o.dtype, device=o.device) for _ in range(world)]
    lb = [torch.empty(rows, dtype=lse.dtype, device=lse.device) for _ in range(world)]
    dist.all_gather(ob, o.reshape(rows, d).contiguous(), group=group)
    dist.all_gather(lb, lse.reshape(rows).contiguous(), group=group)
    return torch.stack(ob), torch.stack(lb)


@dataclass
class SeqShard:
    """One rank's share of a sequence-split layer (B = 1)."""
    rank: int
    world: int
    ranges: List[Tuple[int, int]]
    global_layer: object   # dynsplit.PagedLayer with the global plan (no pages)
    local_layer: object    # dynsplit.PagedLayer over the local tokens/pages


def global_plan(tokens, delim_ids, cfg, static_w10, Hq: int, Hkv: int, world: int):
    """The DD-Select plan of the whole sequence (identical on every rank) and
    the per-rank block ranges."""
    from . import dynsplit as D
    glob = D.build_blocks(tokens, delim_ids, None, None, cfg, static_w10=static_w10, Hq=Hq, Hkv=Hkv)
    nb = int(glob.n_blocks[0])
    return glob, seq_split_ranges(glob.block_starts[0].tolist(), nb, world)


def build_seq_shard(glob, ranges, rank: int, K_local, V_local, cfg, Hq: int):
    """The rank's local pages/digests for its block range (plan given).

    K_local/V_local: [1, S_local, Hkv, d] = the rank's token range
    `shard_token_range(...)` of the layer's K/V.
    """
    from . import dynsplit as D
    world = len(ranges)
    lo, hi = ranges[rank]
    S_loc = int(glob.block_starts[0, hi]) - int(glob.block_starts[0, lo])
    mb_loc = D.max_blocks(max(S_loc, 1), cfg)
    bs_loc, _, _ = local_plan(glob.block_starts[0], lo, hi, mb_loc)
    bs_loc = bs_loc[None].contiguous()
    nb_loc = torch.tensor([hi - lo], dtype=torch.int32, device=K_local.device)
    pf, pb, pv, npg = D.map_pages(bs_loc, nb_loc, max(S_loc, 1), cfg)
    Kp, Vp, dig = D.repack_digest(K_local, V_local, bs_loc, nb_loc, pf, cfg)
    shape = D.make_shape(1, max(S_loc, 1), Hq, K_local.shape[2], K_local.shape[3], 1,
                         D._dtype_code(K_local))
    loc = D.PagedLayer(shape, cfg, glob.w10, bs_loc, nb_loc, pf, pb, pv, npg, Kp, Vp, dig)
    return SeqShard(rank, world, list(ranges), glob, loc)


def shard_token_range(block_starts_row, ranges, rank) -> Tuple[int, int]:
    lo, hi = ranges[rank]
    return int(block_starts_row[lo]), int(block_starts_row[hi])


def shard_scores(q, shard: SeqShard):
    """a5 on the rank's local digests."""
    from . import dynsplit as D
    return D.score_blocks(q, shard.local_layer)


def shard_attend(q, shard: SeqShard, global_scores, budget: int):
    """a6 (global selection, local worklist) + a7 on the rank's pages."""
    from . import dynsplit as D
    Hq = q.shape[1]
    lo, hi = shard.ranges[shard.rank]
    n_glob = int(shard.global_layer.n_blocks[0])
    mb_glob = D.max_blocks(shard.global_layer.shape.S, shard.global_layer.cfg)
    scores = torch.full((1, Hq, mb_glob), float("-inf"), dtype=torch.float32, device=q.device)
    scores[..., :n_glob] = global_scores[..., :n_glob]
    sel = D.select_from_scores(scores, shard.global_layer, budget, Hq, blk_lo=lo, blk_hi=hi)
    o, lse = D.decode_attn(q, shard.local_layer, sel.worklist)
    return o, lse, sel


def seq_split_decode(q, shard: SeqShard, budget: int, group=None):
    """One decode step of one layer under the sequence split (rows a5-a8),
    collectives through torch.distributed (NCCL on GPUs)."""
    from . import dynsplit as D
    Hq = q.shape[1]
    n_glob = int(shard.global_layer.n_blocks[0])
    local_scores = shard_scores(q, shard)                                      # a5 (local)
    global_scores = gather_block_scores(local_scores, shard.ranges, n_glob, group)
    o, lse, sel = shard_attend(q, shard, global_scores, budget)               # a6 + a7
    o_all, lse_all = gather_partials(o, lse, group)
    o_m, lse_m = D.merge_partials(o_all.contiguous(), lse_all.contiguous())  # a8 (rank order)
    return o_m.view(1, Hq, -1), lse_m.view(1, Hq), sel

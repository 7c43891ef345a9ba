"""Multi-GPU plumbing for the DynSplit-KV hot path (torch.distributed).

Two partitions:

* Batch / KV-group partition (BASELINE config 3): each rank owns whole
  sequences, runs the single-GPU path on them, and nothing crosses the
  interconnect on the data path.  `batch_shard` gives a rank's sequences.

* Sequence split (config 4, "sequence-split across 2/4/8 B200 with NCCL LSE
  merge"): every rank holds the global DD-Select plan (block boundaries are a
  cheap function of the tokens) and the pages and digests of a contiguous
  range of blocks.  Per decode step and layer (`SeqSplitDecoder.step`):
    1. local block scores (a5) on the local digests, written straight into the
       rank's all-gather send buffer;
    2. one all-gather of the scores; a fixed index map (built once) places
       every rank's scores at their global block positions, so every rank
       holds the identical global score vector and the budgeted top-k (a6) is
       global and bit-identical on all ranks (block scores do not depend on
       how blocks are split across CTAs or ranks); the worklist keeps only
       the local pages;
    3. local split-K attention (a7) -> (o_r, lse_r); a rank with nothing
       selected for a head yields lse = -inf, o = 0;
    4. all-gather of (o_r, lse_r) and the log-sum-exp merge (a8) in rank order
       (`dynsplit_merge_partials`).
  Every buffer is allocated once, nothing reads device values on the host,
  so a step (all layers) is CUDA-graph capturable with NCCL collectives.

All arithmetic of the method runs in libdynsplit kernels; this module only
moves tensors (collectives, one index gather) and slices plans.  The
collective helpers take plain tensors so they are tested with the gloo
backend on CPU (tests/test_parallel_gloo.py) and, with the library, by two
processes sharing one GPU (tests/test_gpu_seqsplit.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

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


# ---------------------------------------------------------------------------
# collectives (plain tensors; NCCL on GPUs, gloo on CPU and in the
# two-processes-on-one-GPU test)
# ---------------------------------------------------------------------------
def _backend(group=None) -> str:
    return str(dist.get_backend(group)).lower()


def all_gather_flat(out: torch.Tensor, inp: torch.Tensor, group=None) -> None:
    """out[r * n:(r + 1) * n] = rank r's `inp` (n = inp.numel()), in place.
    NCCL: one all_gather_into_tensor (graph-capturable).  gloo: all_gather
    into views of `out` (CUDA tensors are staged through host memory, which
    gloo needs; used by tests only)."""
    world = dist.get_world_size(group)
    n = inp.numel()
    assert out.numel() == world * n
    if _backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp.reshape(-1), group=group)
        return
    if inp.is_cuda:
        host = torch.empty(world * n, dtype=inp.dtype)
        dist.all_gather(list(host.chunk(world)), inp.reshape(-1).cpu(), group=group)
        out.copy_(host.to(out.device))
        return
    dist.all_gather(list(out.reshape(-1).chunk(world)), inp.reshape(-1).contiguous(), group=group)


def score_index(ranges: Sequence[Tuple[int, int]], strides: Sequence[int], Hq: int, send_len: int,
                mb_glob: int) -> torch.Tensor:
    """Index map of the score all-gather.  Rank r's a5 writes head h, local
    block i at send[h * strides[r] + i]; after the all-gather that element is
    at r * send_len + h * strides[r] + i of the gathered buffer.  Returns the
    int64 [Hq * mb_glob] positions of global block (h, lo_r + i); blocks past
    the sequence point at the extra element world * send_len (kept -inf)."""
    world = len(ranges)
    idx = torch.full((Hq, mb_glob), world * send_len, dtype=torch.int64)
    for r, (lo, hi) in enumerate(ranges):
        if hi > lo:
            i = torch.arange(hi - lo, dtype=torch.int64)
            for h in range(Hq):
                idx[h, lo:hi] = r * send_len + h * strides[r] + i
    return idx.reshape(-1)


def gather_global_scores(send: torch.Tensor, gathered: torch.Tensor, idx: torch.Tensor, out: torch.Tensor,
                         group=None) -> None:
    """All-gather every rank's local block scores (`send`, flat) into
    `gathered` (flat, world * send.numel() + 1 elements, the last one -inf)
    and place them at their global positions: out.view(-1) = gathered[idx].
    Every rank ends with bit-identical global scores (exact copies)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n = send.numel()
    if world == 1:
        gathered[:n].copy_(send.reshape(-1))
    else:
        all_gather_flat(gathered[: world * n], send, group)
    torch.index_select(gathered, 0, idx, out=out.view(-1))


# ---- older list-based helpers (kept for the CPU gloo tests of the plumbing)
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
    ob = torch.empty(world * rows * d, dtype=o.dtype, device=o.device)
    lb = torch.empty(world * rows, dtype=lse.dtype, device=lse.device)
    all_gather_flat(ob, o.reshape(-1).contiguous(), group)
    all_gather_flat(lb, lse.reshape(-1).contiguous(), group)
    return ob.view(world, rows, d), lb.view(world, rows)


# ---------------------------------------------------------------------------
# sequence split through the library
# ---------------------------------------------------------------------------
def global_plan(tokens, delim_ids, cfg, static_w10, Hq: int, Hkv: int, world: int):
    """The DD-Select plan of the whole sequence (identical on every rank) and
    the per-rank block ranges (one host read of the plan, at setup)."""
    from . import dynsplit as D
    glob = D.build_blocks(tokens, delim_ids, None, None, cfg, static_w10=static_w10, Hq=Hq, Hkv=Hkv)
    nb = int(glob.n_blocks[0])
    return glob, seq_split_ranges(glob.block_starts[0].tolist(), nb, world)


def shard_token_range(block_starts_row, ranges, rank) -> Tuple[int, int]:
    lo, hi = ranges[rank]
    return int(block_starts_row[lo]), int(block_starts_row[hi])


def local_layer(glob, ranges, rank: int, K_local, V_local, cfg, Hq: int):
    """The rank's local pages/digests for its block range (plan given).
    K_local/V_local: [1, S_local, Hkv, d] = the rank's token range
    (`shard_token_range`) of the layer's K/V."""
    from . import dynsplit as D
    lo, hi = ranges[rank]
    S_loc = max(int(glob.block_starts[0, hi]) - int(glob.block_starts[0, lo]), 1)
    mb_loc = D.max_blocks(S_loc, cfg)
    bs_loc, _, _ = local_plan(glob.block_starts[0], lo, hi, mb_loc)
    bs_loc = bs_loc[None].contiguous()
    nb_loc = torch.tensor([hi - lo], dtype=torch.int32, device=K_local.device)
    pf, pb, pv, npg = D.map_pages(bs_loc, nb_loc, S_loc, cfg)
    Kp, Vp, dig = D.repack_digest(K_local, V_local, bs_loc, nb_loc, pf, cfg)
    shape = D.make_shape(1, S_loc, Hq, K_local.shape[2], K_local.shape[3], 1, D._dtype_code(K_local))
    return D.PagedLayer(shape, cfg, glob.w10, bs_loc, nb_loc, pf, pb, pv, npg, Kp, Vp, dig)


def local_token_counts(glob, ranges) -> List[int]:
    bs = glob.block_starts[0].tolist()
    return [max(bs[hi] - bs[lo], 1) for lo, hi in ranges]


class SeqSplitDecoder:
    """One rank's sequence-split decode of a layer (B = 1), all buffers
    preallocated at construction; `step` launches a5, the score all-gather,
    the index gather, a6, a7 and the partial all-gathers + a8, with no host
    synchronisation (graph-capturable; one decoder can serve every layer of
    a model since the plan is per sequence)."""

    def __init__(self, glob, ranges, rank: int, Hq: int, budget: int, device, group=None):
        from . import dynsplit as D
        self.D = D
        self.glob, self.ranges, self.rank, self.group = glob, list(ranges), rank, group
        self.world = len(ranges)
        self.Hq, self.budget = Hq, budget
        cfg = glob.cfg
        self.cfg = cfg
        self.lo, self.hi = ranges[rank]
        s_locs = local_token_counts(glob, ranges)
        strides = [D.max_blocks(s, cfg) for s in s_locs]           # every rank's a5 row stride
        self.stride = strides[rank]
        send_len = Hq * max(strides)
        self.send = torch.empty(send_len, dtype=torch.float32, device=device)
        self.gathered = torch.full((self.world * send_len + 1,), float("-inf"), dtype=torch.float32,
                                   device=device)
        mb_glob = D.max_blocks(glob.shape.S, cfg)
        self.idx = score_index(self.ranges, strides, Hq, send_len, mb_glob).to(device)
        self.scores = torch.empty(1, Hq, mb_glob, dtype=torch.float32, device=device)
        gshape = D.make_shape(1, glob.shape.S, Hq, glob.shape.Hkv, 128, 1, glob.shape.kv_dtype)
        self.gshape = gshape
        _, ns, mg, kp, wl = D._sel_outputs(gshape, cfg, budget, device, want_blocks=False)
        self.sel_out = (None, ns, mg, kp, wl)
        self.ws_sel = torch.zeros(D.workspace_bytes(D.OP_SELECT, gshape, cfg, budget), dtype=torch.uint8,
                                  device=device)
        self.ws_dec = None
        d = 128
        self.o_part = torch.empty(1, Hq, d, dtype=torch.float32, device=device)
        self.lse_part = torch.empty(1, Hq, dtype=torch.float32, device=device)
        self.o_all = torch.empty(self.world * Hq * d, dtype=torch.float32, device=device)
        self.lse_all = torch.empty(self.world * Hq, dtype=torch.float32, device=device)
        self.o = torch.empty(Hq, d, dtype=torch.float32, device=device)
        self.lse = torch.empty(Hq, dtype=torch.float32, device=device)

    def step(self, q, layer, o=None, lse=None):
        """One layer: q [1, Hq, d] (identical on every rank), `layer` = this
        rank's local PagedLayer.  Returns the merged (o [Hq, d], lse [Hq])
        (written into o / lse when given)."""
        D = self.D
        Hq = self.Hq
        if self.ws_dec is None:
            shp = D._decode_shape(q, layer)
            self.ws_dec = torch.zeros(D.workspace_bytes(D.OP_DECODE_ATTN, shp, layer.cfg), dtype=torch.uint8,
                                      device=q.device)
        # a5 on the local digests, straight into the send buffer (row stride = this rank's)
        D.score_blocks(q, layer, out=self.send[: Hq * self.stride].view(1, Hq, self.stride))
        gather_global_scores(self.send, self.gathered, self.idx, self.scores, self.group)
        # a6: global selection, worklist of the local pages only
        sel = D.select_from_scores(self.scores, self.glob, self.budget, Hq, blk_lo=self.lo, blk_hi=self.hi,
                                   out=self.sel_out, ws=self.ws_sel)
        # a7 on the local pages
        D.decode_attn(q, layer, sel.worklist, out=(self.o_part, self.lse_part), ws=self.ws_dec)
        o = self.o if o is None else o
        lse = self.lse if lse is None else lse
        if self.world == 1:
            o.copy_(self.o_part.view(Hq, -1))
            lse.copy_(self.lse_part.view(Hq))
            return o, lse
        all_gather_flat(self.o_all, self.o_part, self.group)
        all_gather_flat(self.lse_all, self.lse_part, self.group)
        # a8: rank-ordered log-sum-exp merge
        D.merge_partials(self.o_all.view(self.world, Hq, -1), self.lse_all.view(self.world, Hq), out=(o, lse))
        return o, lse

    def selection(self):
        """(n_sel, marginal_block, marginal_keep) of the last step (global, identical on every rank)."""
        return self.sel_out[1], self.sel_out[2], self.sel_out[3]

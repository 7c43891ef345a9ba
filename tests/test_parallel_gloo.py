"""World-size-2 gloo tests (CPU) of the multi-GPU plumbing in
paper_2602_03184_b200/parallel.py.  The per-rank compute is played by the
oracle; what is under test is the sharding, the all-gathers, the global
assembly of block scores and the rank-ordered merge: the sequence-split
result must equal the single-process result (selection exactly, attention to
1e-12)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dynsplit_oracle as O
from paper_2602_03184_b200 import parallel as PAR
from synth import generators as G


def test_batch_shard_partitions():
    for n in range(0, 20):
        for world in (1, 2, 3, 8):
            parts = [PAR.batch_shard(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1


def test_seq_split_ranges_cover_and_balance():
    toks = G.tokens(3, 20000)
    starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
    nb = len(starts) - 1
    for world in (1, 2, 3, 4, 8):
        rs = PAR.seq_split_ranges(starts, nb, world)
        assert rs[0][0] == 0 and rs[-1][1] == nb
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        for r, (lo, hi) in enumerate(rs):
            tok_lo, tok_hi = starts[lo], starts[hi]
            assert abs(tok_lo - r * 20000 / world) <= 46 and abs(tok_hi - (r + 1) * 20000 / world) <= 46


def test_local_plan_shift():
    bs = torch.tensor([0, 20, 55, 80, 100, 100], dtype=torch.int32)
    out, base, s_loc = PAR.local_plan(bs, 1, 3, 6)
    assert base == 20 and s_loc == 60
    assert out.tolist() == [0, 35, 60, 60, 60, 60, 60]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, Hq, Hkv, d, budget = 3000, 8, 2, 32, 300
        g = Hq // Hkv
        toks = G.tokens(21, S)
        q, K, V = G.decode_qkv(22, S, Hq, Hkv, d)
        starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
        nb = len(starts) - 1
        ranges = PAR.seq_split_ranges(starts, nb, world)
        lo, hi = ranges[rank]
        t_lo, t_hi = starts[lo], starts[hi]
        # a5 on the local digests (oracle stands in for the kernel)
        kmax, kmin = O.digests(K[t_lo:t_hi], [s - t_lo for s in starts[lo:hi + 1]])
        local = np.stack([O.block_scores(q[h], kmax[h // g], kmin[h // g]) for h in range(Hq)])
        local_t = torch.zeros(1, Hq, max(hi - lo, 1), dtype=torch.float64)
        local_t[0, :, : hi - lo] = torch.from_numpy(local)
        glob = PAR.gather_block_scores(local_t, ranges, nb).numpy()[0]
        # a6 global selection, a7 on the local tokens only
        o_loc = np.zeros((Hq, d))
        l_loc = np.full(Hq, -np.inf)
        sel = []
        for h in range(Hq):
            toks_sel = O.select_tokens(glob[h], starts, budget)
            sel.append(toks_sel)
            mine = toks_sel[(toks_sel >= t_lo) & (toks_sel < t_hi)]
            if mine.size:
                o_loc[h], l_loc[h] = O.sparse_attention(q[h], K[:, h // g], V[:, h // g], mine,
                                                        1 / math.sqrt(d))
        o_all, l_all = PAR.gather_partials(torch.from_numpy(o_loc), torch.from_numpy(l_loc))
        merged = [O.merge_partials(o_all[:, h].numpy(), l_all[:, h].numpy()) for h in range(Hq)]
        ref = O.decode_step(q, K, V, starts, budget)
        ok = True
        for h in range(Hq):
            ok &= np.array_equal(sel[h], ref["tokens"][h])
            ok &= np.allclose(merged[h][0], ref["o"][h], atol=1e-12)
            ok &= abs(merged[h][1] - ref["lse"][h]) < 1e-12
        ok &= np.array_equal(glob, np.stack(ref["scores"]))
        out_q.put((rank, bool(ok), ranges))
    finally:
        dist.destroy_process_group()


def test_seq_split_world2_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert res[0][2] == res[1][2]


def _worker_index(rank, world, port, out_q):
    """score_index + gather_global_scores: every rank writes its local block
    scores with its own row stride into its send buffer; after the gather each
    global (head, block) must hold exactly that rank's value, blocks past the
    sequence -inf, identical on every rank."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        toks = G.tokens(41, 9000)
        starts = O.segment(toks, G.T7_IDS, G.T7_W10, 32, 14)
        nb = len(starts) - 1
        ranges = PAR.seq_split_ranges(starts, nb, world)
        Hq, mb_glob = 5, nb + 7
        strides = [max(1, (starts[hi] - starts[lo]) // 18 + 1) for lo, hi in ranges]
        send_len = Hq * max(strides)
        idx = PAR.score_index(ranges, strides, Hq, send_len, mb_glob)
        # the "true" global scores: value = 1000 h + block + 0.25
        truth = np.full((Hq, mb_glob), -np.inf)
        for h in range(Hq):
            truth[h, :nb] = 1000 * h + np.arange(nb) + 0.25
        lo, hi = ranges[rank]
        send = torch.full((send_len,), 7.5, dtype=torch.float64)     # junk beyond the rank's blocks
        for h in range(Hq):
            send[h * strides[rank]: h * strides[rank] + hi - lo] = torch.from_numpy(truth[h, lo:hi])
        gathered = torch.full((world * send_len + 1,), float("-inf"), dtype=torch.float64)
        out = torch.empty(Hq, mb_glob, dtype=torch.float64)
        PAR.gather_global_scores(send, gathered, idx, out)
        out_q.put((rank, bool(np.array_equal(out.numpy(), truth))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_score_index_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_index, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res

"""Multi-rank α-grid host logic on CPU (gloo, world size 2): LPT sharding covers every
chain exactly once, each rank reduces only its chains, the all-gather + argmax gives
every rank the same α* as a single process (the grid search is
parallel over independent replays)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import tracegen as tg
from paper_2411_19379_b200 import grid as G


def _workload():
    w = tg.workload(3, R=1500)
    w.alphas = (0.0, 1 / 16, 0.5, 2.0, 64.0)
    w.n_segments = 5
    return w


def _chain_sums(w, chain_ids):
    """Per-(variant, α) hit sums of the given chains, computed by the CPU oracle
    (test stand-in for the device replay, which needs a GPU)."""
    import oracle as O
    segs = w.segments()
    na, ns = len(w.alphas), len(segs)
    snaps, *_ = O.live_pass(w.trace, w.variants[0], w.window)
    chains = []
    for c in chain_ids:
        a, s = (c // ns) % na, c % ns
        chains.append((0, w.alphas[a], segs[s][0], segs[s][1], s))
    out = np.zeros((1, na), np.int64)
    if chains:
        _, _, _, hs, _ = O.run_chains(w.trace, w.variants, chains, snaps, n_threads=2)
        for c, x in zip(chain_ids, hs):
            out[0, (c // ns) % na] += int(x)
    return out


def test_lpt_shard_partitions_and_balances():
    costs = np.random.default_rng(0).integers(100, 10_000, 16 * 128)
    for world in (1, 2, 4, 8):
        sh = G.lpt_shard(costs, 128, 16, world)
        allc = np.concatenate(sh)
        assert sorted(allc.tolist()) == list(range(len(costs)))
        loads = [costs[s.astype(np.int64)].sum() for s in sh]
        assert max(loads) - min(loads) <= costs.max()
        assert [x.tolist() for x in G.lpt_shard(costs, 128, 16, world)] == [x.tolist() for x in sh]


def _worker(rank, world, port, res):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    w = _workload()
    lens = w.trace.lin.astype(np.int64) + w.trace.lout
    segs = [(f, n, k) for k, (f, n) in enumerate(w.segments())]
    costs = G.chain_costs(lens, segs, 1, len(w.alphas))
    shard = G.lpt_shard(costs, len(segs), len(w.alphas), world)[rank]
    part = torch.from_numpy(_chain_sums(w, shard.tolist()))
    tot = G.gather_hit_sums(part, world)
    res[rank] = (tot.numpy().tolist(), G.select_alpha(w.alphas, tot.numpy()))
    torch.distributed.destroy_process_group()


def test_two_ranks_gloo_select_same_alpha():
    w = _workload()
    total = len(w.alphas) * len(w.segments())
    single = _chain_sums(w, list(range(total)))
    want = G.select_alpha(w.alphas, single)
    mgr = mp.Manager()
    res = mgr.dict()
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(2, port, res), nprocs=2, join=True)
    assert res[0] == res[1]
    assert res[0][0] == single.tolist()
    assert res[0][1] == want
